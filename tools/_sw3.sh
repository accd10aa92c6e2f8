mkdir -p gpurun_out/sw3
timeout 1800 python tools/c3_sweep.py gpurun_out/sw3/sweep770.csv 7 770 > gpurun_out/sw3/sweep770.log 2>&1
timeout 1500 python tools/c3_sweep.py gpurun_out/sw3/sweep_full.csv 5 0 > gpurun_out/sw3/sweep_full.log 2>&1
