run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['list_rebuild_groups'],d['h_iters'])")"; }
run default
run static SPH_WALK_STATIC=1
run head SPH_LIB=paper_1404_2303_b200/libsph_head.so
run default2
run static2 SPH_WALK_STATIC=1
run head2 SPH_LIB=paper_1404_2303_b200/libsph_head.so
