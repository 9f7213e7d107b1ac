#!/bin/bash
# Sweep tile configurations of one op: tools/sweep.sh fwd_c "fwd collapsed 0"
op=$1; shift
for cfg in 128,64,256,4,1 128,64,256,2,1 128,32,256,4,1 128,32,256,2,1 64,64,128,4,1 64,64,128,2,1 64,32,128,4,1 32,32,64,4,1 32,32,64,1,1 64,64,128,1,1 128,32,256,1,1 128,64,256,1,1; do
  echo -n "$cfg: "; env LFM_FORCE_$op=$cfg python tools/prof_op.py $@ 3 2>&1 | tail -1
done
