run() { local name=$1; local cfg=$2; shift; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['groups'],d['cells'],d['h_iters'])")"; }
run default '{}'
for v in "$@"; do run $v '{}' SPH_LIB=paper_1404_2303_b200/libsph_$v.so; done
run default2 '{}'
