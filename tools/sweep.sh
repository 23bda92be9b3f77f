#!/bin/bash
run() { local name=$1; shift; local cfg=$1; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2),'kd',round(d['ms_kernel_density_full'],3),'kf',round(d['ms_kernel_force'],3),d['groups'],d['cells'],d['list_dens'])")"; }
run s32 '{"split_count": 32, "split_fraction": 0.0}'
run s64_sort32 '{"split_count": 64, "split_fraction": 0.0, "sort_min_len": 32}'
run s64_nosort '{"split_count": 64, "split_fraction": 0.0, "sort_min_len": 100000}'
run s128_sort32 '{"split_count": 128, "split_fraction": 0.0, "sort_min_len": 32}'
run paper '{"split_count": 300, "split_fraction": 0.875}'
run paper_sort0 '{"split_count": 300, "split_fraction": 0.875, "sort_min_len": 0}'
run paper_nosort '{"split_count": 300, "split_fraction": 0.875, "sort_min_len": 100000}'
