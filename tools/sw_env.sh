run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['list_rebuild_groups'],d['h_iters'])")"; }
run default
run cm130 SPH_COLD_MARGIN=1.3
run cm135 SPH_COLD_MARGIN=1.35
run cm125 SPH_COLD_MARGIN=1.25
run cm140 SPH_COLD_MARGIN=1.4
run default2
