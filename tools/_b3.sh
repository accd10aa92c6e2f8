mkdir -p gpurun_out/b3
for c in cfg2 cfg3 cfg4; do timeout 600 python bench.py --config $c > gpurun_out/b3/bench_$c.json 2> gpurun_out/b3/bench_$c.err; done
