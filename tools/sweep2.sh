#!/bin/bash
# tools/sweep2.sh OP "cfg1 cfg2 ..." prof_op args...
op=$1; cfgs=$2; shift 2
for cfg in $cfgs; do echo -n "$op $cfg: "; env LFM_FORCE_$op=$cfg python tools/prof_op.py $@ 3 2>&1 | tail -1; done
