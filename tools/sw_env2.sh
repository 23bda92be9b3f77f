run() { local name=$1; local cfg=$2; shift; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2))")"; }
run default '{}'
run take48 '{}' SPH_LIB=paper_1404_2303_b200/libsph_take48.so
run take96 '{}' SPH_LIB=paper_1404_2303_b200/libsph_take96.so
run s40 '{"split_count": 40}'
run s56 '{"split_count": 56}'
run cm09 '{}' SPH_COLD_MARGIN=0.9
run cm11 '{}' SPH_COLD_MARGIN=1.1
run rm105 '{}' SPH_REGROW_MARGIN=1.05
run rm12 '{}' SPH_REGROW_MARGIN=1.2
run default2 '{}'
