#!/usr/bin/env bash
# Multi-GPU validation for a box with >= 2 GPUs (none of this round's gpurun
# calls had more than one): the two-process parity tests on distinct GPUs
# (NVLink peers; tests/test_multiprocess_gpu.py takes a GPU per rank when it
# can), bench.py over torchrun at every world size the box allows, and the
# NVLink counters of the push kernels (tools/ncu_nvlink.sh).
#   usage: bash tools/multigpu_check.sh OUT_DIR
set -u
OUT=${1:-gpurun_out/multigpu}
mkdir -p "$OUT"
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG" | tee "$OUT/summary.txt"
timeout 900 python -m pytest tests/test_multiprocess_gpu.py -q > "$OUT/pytest_multiprocess.log" 2>&1
echo "multiprocess tests rc=$? $(tail -1 "$OUT/pytest_multiprocess.log")" | tee -a "$OUT/summary.txt"
for n in 2 4 8; do
  [ "$n" -le "$NG" ] || continue
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
    --master-port $((29600 + n)) bench.py --gpus "$n" > "$OUT/bench_n$n.json" 2> "$OUT/bench_n$n.err"
  echo "bench n=$n rc=$? $(tail -c 300 "$OUT/bench_n$n.json")" | tee -a "$OUT/summary.txt"
done
if [ "$NG" -ge 2 ]; then
  timeout 1200 bash tools/ncu_nvlink.sh 2 "$OUT/ncu_nvlink_n2" > "$OUT/ncu_nvlink.log" 2>&1
  echo "ncu nvlink rc=$?" | tee -a "$OUT/summary.txt"
fi
