# session 3, call r: pivot-column timers (HPS_PROF_PIVOT=1 diagnostics build) at p = 8 / 12 / 16
O=gpurun_out/${OUT:-s3r}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for p in 8 12 16; do
  n=$([ $p = 8 ] && echo 5920 || ([ $p = 12 ] && echo 2960 || echo 592))
  HPS_LIB=$L/libhps_leaf_profpiv.so timeout 300 python tools/prof_breakdown.py --p $p --leaves $n > $O/prof${p}_piv.txt 2>&1
done
