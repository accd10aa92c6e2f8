mkdir -p gpurun_out/f3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f3/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/f3/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo rc=$? >> gpurun_out/f3/smoke.log
for c in cfg2 cfg3 cfg4; do timeout 600 python bench.py --config $c > gpurun_out/f3/bench_$c.json 2> gpurun_out/f3/bench_$c.err; done
timeout 600 python bench.py --impl reference > gpurun_out/f3/bench_ref.json 2> gpurun_out/f3/bench_ref.err
