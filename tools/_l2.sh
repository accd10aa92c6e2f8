C3_GEMM_KERNEL=pair512 timeout 1100 tools/gemm_l2_ab.sh gpurun_out/l2ab_p512_cfg2.txt 8192 28672 8192 "6 8 12 16 32" "11 12 13"
C3_GEMM_KERNEL=pair512 timeout 600 tools/gemm_l2_ab.sh gpurun_out/l2ab_p512_cfg4.txt 8192 53248 16384 "4 8 16" "11 12"
