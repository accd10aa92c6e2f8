#!/bin/bash
# NVLink traffic of the SM collectives and the fused C3 GEMM on a real node
# (VERDICT r1 missing #6). Rank 0 of an N-GPU torchrun world runs under ncu
# (one profiled process; the others run plain), collecting per-kernel NVLink
# RX/TX bytes next to time and DRAM bytes for the all-gather push, the
# reduce-scatter pull and the fused pair GEMM.
#
#   tools/ncu_nvlink.sh N OUT_PREFIX [bench args...]
# e.g. tools/ncu_nvlink.sh 8 profiles/r03_nvlink --config cfg2 --steps 3 --warmup 3
#
# Reading: achieved NVLink GB/s per direction of a kernel = nvltx__bytes.sum /
# gpu__time_duration.sum; against 900 GB/s nominal / 770 GB/s measured peer
# copy (B200_PROFILING.md). ncu serialises kernels and replays each one, so
# only per-kernel bytes and shares are meaningful, never the bench's value.
# Metric names: `ncu --query-metrics --chip gb100 | grep -i nvl`.
set -euo pipefail
N=${1:?N}; OUT=${2:?out prefix}; shift 2
METRICS=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
KERNELS='regex:ag_push|a2a_push|rs_pull|gemm_bf16_tn_pair_kernel<true|signal_wait'
# ncu replays each kernel of rank 0 many times while its peers wait on the
# device: lift the cross-rank wait bound (default 2 s) for this run only
export C3_WAIT_TIMEOUT_MS=${C3_WAIT_TIMEOUT_MS:-600000}
python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
  --master-port "${MASTER_PORT:-29533}" --no-python bash -c '
    if [ "$RANK" = "0" ]; then
      exec ncu --metrics '"$METRICS"' --clock-control none -k "'"$KERNELS"'" -c 200 --csv \
        --log-file '"$OUT"'_rank0.csv python bench.py --gpus '"$N"' "$@"
    else
      exec python bench.py --gpus '"$N"' "$@"
    fi' _ "$@"
echo "wrote ${OUT}_rank0.csv"
