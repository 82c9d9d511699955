#!/bin/bash
for lib in nopdl pdl1 default; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none -k regex:"block_" -c 8 --csv python tools/scores_dump.py /tmp/x.npz 2>/dev/null | grep "gpu__time" | awk -F'","' '{print $5":"$NF}' | tr -d '"' | sed 's/(.*)//' | tr '\n' ' ' | sed "s/^/$lib /"; echo
done
