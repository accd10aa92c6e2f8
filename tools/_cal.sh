mkdir -p gpurun_out/cal
timeout 900 python tools/calibrate_b200.py gpurun_out/cal > gpurun_out/cal/calibrate.log 2>&1
ls gpurun_out/cal >> gpurun_out/cal/calibrate.log
cp gpurun_out/cal/*slowdown-tables.csv data/b200-loopback-slowdown-tables.csv 2>/dev/null
timeout 1500 python tools/c3_sweep.py gpurun_out/cal/sweep770.csv 7 770 > gpurun_out/cal/sweep770.log 2>&1
timeout 1500 python tools/c3_sweep.py gpurun_out/cal/sweep_full.csv 5 0 > gpurun_out/cal/sweep_full.log 2>&1
