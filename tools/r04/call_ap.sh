# session 3, call ap: run-to-run determinism at p = 20 (300 leaves), 30 runs: the session-start kernel (08dcea8) and the pre-defer kernel
O=gpurun_out/${OUT:-s3ap}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for v in start defer0; do
  HPS_LIB=$L/libhps_leaf_$v.so timeout 1200 python tools/r04/determinism.py 20 300 30 >> $O/det.jsonl 2>> $O/det.err
done
