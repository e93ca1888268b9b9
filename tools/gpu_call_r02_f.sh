# round 2: per-op breakdown with one CTA per SM (no co-resident GEMM) vs two
O=gpurun_out/${OUT:-r2f}; mkdir -p $O
HPS_DEBUG=8 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 296 > $O/prof_p16_onecta.txt 2>&1
cat $O/prof_p16_onecta.txt
