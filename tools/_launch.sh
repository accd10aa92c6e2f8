mkdir -p gpurun_out/fin3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/fin3/launches.csv python bench.py --steps 3 --warmup 3 --strategy c3_base --strategies c3_base,c3_sp,conccl,conccl_rp --no-cpu-baseline > gpurun_out/fin3/bench_ncu.json 2> gpurun_out/fin3/bench_ncu.err
echo rc=$? >> gpurun_out/fin3/bench_ncu.err
