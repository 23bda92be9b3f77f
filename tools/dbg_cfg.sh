#!/bin/bash
# usage: tools/dbg_cfg.sh CONFIG [nsample]
SPH_DEBUG=1 timeout 600 python tools/dbg_run.py "$@"
