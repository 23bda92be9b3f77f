#!/bin/bash
# C4 timing sweep over tuning env vars: one line per variant (warm, no debug timers)
run() { local name=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),d['list_rebuild_groups'])")"; }
for rm in 1.05 1.1 1.15 1.2; do run rm$rm SPH_REGROW_MARGIN=$rm; done
for cm in 1.1 1.2 1.3; do run cm${cm}_rm1.1 SPH_COLD_MARGIN=$cm SPH_REGROW_MARGIN=1.1; done
