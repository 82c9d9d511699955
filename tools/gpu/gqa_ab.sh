#!/bin/bash
# GQA dK/dV pair order A/B (alt_lib/qmajor.so vs alt_lib/headmajor.so) at C5 (128K, 32q/8kv),
# plus MHA (32/32) for the DRAM-read comparison: CUDA-event times, then an ncu DRAM launch list.
OUT=gpurun_out/gqa_ab; mkdir -p $OUT
for lib in qmajor headmajor hmpf; do
  SB_LIB_PATH=alt_lib/$lib.so timeout 600 python tools/sweep_c5.py --keeps 0.1,0.3 --reps 5 > $OUT/sweep_$lib.log 2>&1; echo "$lib rc $?"; grep '^{' $OUT/sweep_$lib.log
done
SB_LIB_PATH=alt_lib/hmpf.so timeout 600 python tools/sweep_c5.py --keeps 0.1,0.3 --reps 5 --kv-heads 32 > $OUT/sweep_mha.log 2>&1; echo "mha rc $?"; grep '^{' $OUT/sweep_mha.log
for cfg in "qmajor 8" "headmajor 8" "hmpf 8" "hmpf 32"; do
  set -- $cfg
  SB_LIB_PATH=alt_lib/$1.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"attn_bwd_dkv|attn_bwd_dq|attn_fwd2" -c 14 --csv --log-file $OUT/ncu_$1_$2.csv \
    python tools/sweep_c5.py --keeps 0.1 --reps 1 --kv-heads $2 > $OUT/ncu_$1_$2.log 2>&1; echo "ncu $cfg rc $?"
done
