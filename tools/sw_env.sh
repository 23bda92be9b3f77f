run() { local name=$1; local cfg=$2; shift; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['groups'],d['cells'],d['h_iters'])")"; }
run default '{}'
run cmax1024 '{}' SPH_GROUP_CMAX=1024
run cmax2048 '{}' SPH_GROUP_CMAX=2048
run ucap512 '{}' SPH_UCAP=512
run ucap1024 '{}' SPH_UCAP=1024
run s56 '{"split_count": 56}'
run default2 '{}'
