#!/bin/bash
run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),'kd',round(d['ms_kernel_density_full'],3),'kf',round(d['ms_kernel_force'],3))")"; }
run compact
run simple SPH_FORCE_SIMPLE=1
