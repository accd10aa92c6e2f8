#!/bin/bash
# GEMM L2 A/B (dev aid): raster band x operand L2 policy on one shape.
# For each (band, policy) pair: ncu DRAM bytes of one launch, then interleaved
# event timing against cuBLAS in its own process (tools/gemm_ab.py).
# Usage: tools/gemm_l2_ab.sh OUT M N K "bands" "policies"
OUT=$1; M=$2; N=$3; K=$4; BANDS=${5:-"8 12 16"}; POLS=${6:-"11 13 12 33"}
: > "$OUT"
for b in $BANDS; do for p in $POLS; do
  echo "== band=$b pol=$p" >> "$OUT"
  C3_GEMM_BAND=$b C3_GEMM_POL=$p ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gemm -s 1 -c 1 python tools/ncu_target.py gemm $M $N $K 2>/dev/null \
    | grep -E "dram__|gpu__time" >> "$OUT"
done; done
for r in 1 2; do for b in $BANDS; do for p in $POLS; do
  echo "time band=$b pol=$p $(C3_GEMM_BAND=$b C3_GEMM_POL=$p python tools/gemm_ab.py $M $N $K 15)" >> "$OUT"
done; done; done
