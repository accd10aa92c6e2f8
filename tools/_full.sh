mkdir -p gpurun_out/fin
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/fin/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo rc=$? >> gpurun_out/fin/smoke.log
timeout 600 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fin/bench_ncu.log 2>&1
C3_GEMM_KERNEL=pair512 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -s 1 -c 1 -o gpurun_out/fin/ncu_gemm_pair512_r01 python tools/ncu_target.py gemm 8192 28672 8192 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ag_push -s 2 -c 1 -o gpurun_out/fin/ncu_ag_r01b python tools/ncu_target.py ag > /dev/null 2>&1
