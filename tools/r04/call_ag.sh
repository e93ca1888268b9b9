# session 3, call ag: breakdowns of the new default (GEMM producer phases, pivot columns) at p = 16 and 12
O=gpurun_out/${OUT:-s3ag}; mkdir -p $O
L=paper_2503_04033_b200/_lib
timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16.txt 2>&1
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_gemm.txt 2>&1
HPS_LIB=$L/libhps_leaf_profpiv.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_piv.txt 2>&1
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 12 --leaves 2960 > $O/prof12_gemm.txt 2>&1
