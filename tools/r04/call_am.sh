# session 3, call am: run-to-run determinism at p = 20 (300 leaves: endgame sharing) — HEAD vs the pre-warp-producer kernel
O=gpurun_out/${OUT:-s3am}; mkdir -p $O
L=paper_2503_04033_b200/_lib
timeout 900 python tools/r04/determinism.py 20 300 8 >> $O/det.jsonl 2>> $O/det.err
HPS_LIB=$L/libhps_leaf_wp0.so timeout 900 python tools/r04/determinism.py 20 300 8 >> $O/det.jsonl 2>> $O/det.err
timeout 900 python tools/r04/determinism.py 16 600 6 >> $O/det.jsonl 2>> $O/det.err
HPS_LIB=$L/libhps_leaf_wp0.so timeout 900 python tools/r04/determinism.py 16 600 6 >> $O/det.jsonl 2>> $O/det.err
