#!/bin/bash
# ncu launch list of one bench configuration: tools/gpu/launches.sh OUTDIR "<bench args>"
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python bench.py --profile-only $2 > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --profile-only $2 > $OUT/ncu.log 2>&1; echo "ncu rc $?"
python tools/launch_summary.py $OUT/launches.csv | head -30
