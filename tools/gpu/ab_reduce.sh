#!/bin/bash
# prep launch-shape A/B: bwd_prep kernel time (ncu, C3 profile-only, 4 launches) per library.
for lib in default "$@"; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dkv_split_reduce -c 4 --csv python bench.py --profile-only 2>/dev/null | grep "gpu__time" | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$lib reduce ns: /"; echo
done
unset SB_LIB_PATH
