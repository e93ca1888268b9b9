# session 3, call ao: run-to-run determinism at p = 20 (300 leaves), 30 runs per build
O=gpurun_out/${OUT:-s3ao}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for v in wp0 wb0 op0; do
  HPS_LIB=$L/libhps_leaf_$v.so timeout 1200 python tools/r04/determinism.py 20 300 30 >> $O/det.jsonl 2>> $O/det.err
done
