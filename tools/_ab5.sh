O=gpurun_out/split_ab.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or fused or llama or cap" >> $O 2>&1
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for r in 1 2; do echo "== ncu pair512 round $r" >> $O
  C3_GEMM_KERNEL=pair512 timeout 200 ncu --metrics $M --clock-control none -k regex:gemm -s 1 -c 1 python tools/ncu_target.py gemm 8192 28672 8192 2>/dev/null | grep -E "^\s+(gpu__|sm__|lts__|dram__)" >> $O
done
for sh in "8192 28672 8192" "8192 8192 8192" "8192 53248 16384"; do
  timeout 300 python tools/gemm_variant_ab.py $sh >> $O 2>&1
done
