# round 2: GPU tests after the flush policy change + executed-flop profile of the leaf kernel
O=gpurun_out/${OUT:-r2e}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof_p16.txt 2>&1
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 20 --leaves 296 > $O/prof_p20.txt 2>&1
cat $O/prof_p16.txt
