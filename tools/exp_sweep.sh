#!/bin/bash
# timing experiments on C4 (debug timers), one line per variant
run() { # name, env...
  local name=$1; shift
  env "$@" SPH_DEBUG=1 SPH_DBG_CFG='{"split_count": 64, "split_fraction": 0.0}' timeout 300 python tools/dbg_run.py C4 10 > gpurun_out/exp_$name.log 2>&1
  echo "== $name: $(grep -E 'density kernel' gpurun_out/exp_$name.log | head -4 | awk '{print $4}' | tr '\n' ' ') force: $(grep -E 'force call' gpurun_out/exp_$name.log | awk '{print $4}')"
}
run base
run desc16 SPH_DESC_MIN=16
run desc64 SPH_DESC_MIN=64
run desc128 SPH_DESC_MIN=128
run desc100k SPH_DESC_MIN=100000
run r64 SPH_LIB=build/libsph_r64.so
