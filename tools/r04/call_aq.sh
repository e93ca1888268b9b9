# session 3, call aq: determinism at p = 20 (300 leaves, 30 runs): share-publish fence (HEAD), no fence (sf0), no fence + sharing off
O=gpurun_out/${OUT:-s3aq}; mkdir -p $O
L=paper_2503_04033_b200/_lib
timeout 1200 python tools/r04/determinism.py 20 300 30 >> $O/det.jsonl 2>> $O/det.err
HPS_DEBUG=16 HPS_LIB=$L/libhps_leaf_sf0.so timeout 1200 python tools/r04/determinism.py 20 300 30 >> $O/det.jsonl 2>> $O/det.err
