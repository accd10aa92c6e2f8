M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum"
O=gpurun_out/clk_ab.txt; : > $O
for r in 1 2; do
for w in pair wide cublas; do
  echo "== $w round $r" >> $O
  if [ $w = cublas ]; then t=cublas; k='nvjet'; else t=gemm; k='gemm'; fi
  C3_GEMM_KERNEL=$w ncu --metrics $M --clock-control none -k regex:$k -s 1 -c 1 python tools/ncu_target.py $t 8192 28672 8192 2>/dev/null | grep -E "^\s+(gpu__|sm__|lts__|dram__)" >> $O
done; done
