#!/bin/bash
# A/B of libsph variants (tools/build_variant.sh): a1-a3 at 16.8M (tools/binning_run.py) and the C4 step
for r in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then L=paper_1404_2303_b200/libsph.so; else L=paper_1404_2303_b200/libsph_$v.so; fi
  echo -n "$v "; SPH_LIB=$L python tools/binning_run.py 16777216 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('a1-a3 16.8M', round(d['ms_a1_a3'],3), round(d['frac'],3), end=' ')"
  SPH_LIB=$L timeout 300 python tools/prof_run.py C4 4 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4', round(d['ms_total_events'],3), round(d['ms_build'],3), round(d['ms_density'],3), round(d['ms_force'],3))"
done; done
