#!/bin/bash
# A/B of libsph variants on C4 (bench configuration): NB walk / union walk / step ms, 2 rounds
for r in 1 2; do for n in "$@"; do
  echo -n "$n "; SPH_LIB=paper_1404_2303_b200/libsph_$n.so timeout 300 python tools/prof_run.py C4 4 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_total_events'],3), round(d['ms_build'],3), round(d['ms_density'],3), round(d['ms_force'],3))"
done; done
