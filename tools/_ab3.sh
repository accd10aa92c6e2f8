O=gpurun_out/p512_full.txt; : > $O
timeout 1200 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo rc=$? >> $O
for c in ag a2a rs; do
  timeout 300 python tools/coresident_ab.py $c 770 16,24,32,48,64 >> $O 2>&1
done
timeout 300 python tools/coresident_ab.py ag 0 16,24,32,148 >> $O 2>&1
timeout 120 python tools/comm_ab.py ag 896 24,48,74,148,296 >> $O 2>&1
