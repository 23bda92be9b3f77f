#!/bin/bash
# run dbg_run on several configs with SPH_DEBUG, extra args passed via SPH_DBG_CFG (json kwargs)
for c in "$@"; do SPH_DEBUG=1 timeout 600 python tools/dbg_run.py $c 1000 > gpurun_out/dbg_$c.log 2>&1; echo "$c rc=$?"; done
