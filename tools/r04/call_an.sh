# session 3, call an: run-to-run determinism at p = 20 (300 leaves): one-pass bounds (HEAD) / committed kernel (op0) / warp producer only (wb0)
O=gpurun_out/${OUT:-s3an}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for v in op0 wb0 head; do
  lib=$L/libhps_leaf_$v.so; [ $v = head ] && lib=$L/libhps_leaf.so
  HPS_LIB=$lib timeout 900 python tools/r04/determinism.py 20 300 12 >> $O/det.jsonl 2>> $O/det.err
done
