#!/bin/bash
# cold-start record margin (sph_config.cold_margin) on the bench workload and on C3:
#   bash tools/cold_margin_sweep.sh [configs...]
cfgs=${@:-C4 C3}
for r in 1 2; do for name in $cfgs; do
for cm in 1.1 1.15 1.2 1.25; do
  echo -n "$name cold_margin $cm "; timeout 300 python tools/prof_run.py $name 4 "{\"cold_margin\": $cm}" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_total_events'],3), round(d['ms_build'],3), round(d['ms_density'],3), round(d['ms_force'],3))"
done; done; done
