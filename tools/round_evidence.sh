#!/usr/bin/env bash
# One gpurun call's worth of round-end evidence (B200, one GPU): the GPU test
# suite, smoke(), the default bench line, every BASELINE config in both arms,
# the ncu launch list of a short bench run and an ncu --set full capture of
# the cfg2 pair GEMM. Output under gpurun_out/$TAG/.
#   usage: bash tools/round_evidence.sh TAG
set -u
TAG=${1:-evidence}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/gputest.log" 2>&1; echo "pytest rc=$?"; tail -2 "$OUT/gputest.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "bench rc=$?"
for c in cfg2_448 cfg3 cfg4 cfg4_mb cfg4_mb64 cfg2_a2a cfg1; do
  timeout 900 python bench.py --config $c > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"; echo "bench $c rc=$?"
  timeout 600 python bench.py --config $c --impl reference > "$OUT/bench_${c}_reference.json" 2>> "$OUT/bench_$c.err"
done
timeout 600 python bench.py --impl reference > "$OUT/bench_default_reference.json" 2>> "$OUT/bench_default.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file "$OUT/launches_bench.csv" \
  python bench.py --steps 3 --warmup 3 --no-green --no-cpu-baseline > "$OUT/bench_under_ncu.log" 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tn_pair -s 1 -c 1 \
  -o "$OUT/ncu_gemm_cfg2" python tools/ncu_target.py gemm 8192 28672 8192 > "$OUT/ncu_full.log" 2>&1; echo "ncu full rc=$?"
for tool in memcheck synccheck racecheck; do
  C3_SANITIZE_F32=1 timeout 900 compute-sanitizer --tool $tool python tools/dev/sanitize_target.py > "$OUT/sanitizer_$tool.txt" 2>&1; echo "sanitizer $tool rc=$?"
done
