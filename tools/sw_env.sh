run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['list_rebuild_groups'],d['h_iters'])")"; }
export SPH_LIB=paper_1404_2303_b200/libsph_head.so
run head
run k512 SPH_NBK=512
run k256 SPH_NBK=256
run k192 SPH_NBK=192
run k128 SPH_NBK=128
unset SPH_LIB
run dyn_k256 SPH_NBK=256
run dyn_k128 SPH_NBK=128
