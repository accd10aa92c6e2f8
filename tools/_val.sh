mkdir -p gpurun_out/val
timeout 300 python -m pytest tests/test_gpu_runtime_model.py -q > gpurun_out/val/pytest.log 2>&1
timeout 1500 python tools/c3_sweep.py gpurun_out/val/sweep770.csv 7 770 > gpurun_out/val/sweep770.log 2>&1
timeout 600 python bench.py > gpurun_out/val/bench.json 2> gpurun_out/val/bench.err
timeout 600 python bench.py --config cfg3 > gpurun_out/val/bench_cfg3.json 2> gpurun_out/val/bench_cfg3.err
timeout 600 python bench.py --config cfg4 > gpurun_out/val/bench_cfg4.json 2> gpurun_out/val/bench_cfg4.err
