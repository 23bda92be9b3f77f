#!/bin/bash
run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_total_events'],2),'kd',round(d['ms_kernel_density_full'],3),'kf',round(d['ms_kernel_force'],3))")"; }
run f8s1 SPH_LIB=paper_1404_2303_b200/libsph_f8s1.so
run d1f1 SPH_LIB=paper_1404_2303_b200/libsph_d1f1.so
run w4 SPH_LIB=paper_1404_2303_b200/libsph_w4.so
run w16 SPH_LIB=paper_1404_2303_b200/libsph_w16.so
