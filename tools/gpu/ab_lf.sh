#!/bin/bash
for r in 1 2; do for lib in lead4 lf16; do
  export SB_LIB_PATH=alt_lib/$lib.so
  C2=1 timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dkv per-CTA (us)" | sed "s/^/$lib C2 $r /"
  timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dkv per-CTA (us)" | sed "s/^/$lib C3 $r /"
done; done
for lib in lead4 lf16; do
  export SB_LIB_PATH=alt_lib/$lib.so
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 3 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib C5 /" | cut -c1-200
done
