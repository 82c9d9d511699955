#!/bin/bash
# C2 / C5 kernel times: current lib vs alt_lib/headmajor.so (before the dK/dV split), same box, alternating.
for r in 1 2; do
for lib in default headmajor; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 python tools/time_kernels.py 2>&1 | grep -E "attn_bwd|fwd |split|sort|prep" | sed "s/^/$lib $r C2 /"
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 5 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib $r C5 /" | cut -c1-260
done
done
unset SB_LIB_PATH
