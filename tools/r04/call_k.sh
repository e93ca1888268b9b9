# session 3, call k: GEMM sub-phase profile (HPS_PROF_GEMM=1 diagnostics build) at p=16 and p=20
O=gpurun_out/${OUT:-s3k}; mkdir -p $O
L=paper_2503_04033_b200/_lib
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_gemm.txt 2>&1
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 20 --leaves 296 > $O/prof20_gemm.txt 2>&1
