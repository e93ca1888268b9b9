# session 3, call m: per-op breakdown at p = 12 (configs[1] order) and p = 8 with the GEMM producer diagnostics
O=gpurun_out/${OUT:-s3m}; mkdir -p $O
L=paper_2503_04033_b200/_lib
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 12 --leaves 2960 > $O/prof12_gemm.txt 2>&1
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 8 --leaves 5920 > $O/prof8_gemm.txt 2>&1
