#!/bin/bash
# bwd_prep A/B under ncu (serialized per-kernel durations; PDL makes profiler-event kernel times
# include the wait on the predecessor).
for lib in pdl1 prepA prepB; do
  SB_LIB_PATH=alt_lib/$lib.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"bwd_prep" -c 6 --csv python tools/time_kernels.py 2>/dev/null | grep bwd_prep | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$lib /"; echo
done
