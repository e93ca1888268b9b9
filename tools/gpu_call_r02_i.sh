# round 2: k-chunk 32 x 2 stages, L2 promotion of the TMA maps; base twice for the noise
O=gpurun_out/${OUT:-r2i}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 888 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run kc32s2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_kc32s2.so
run promo128 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_promo128.so
run promo0 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_promo0.so
run red3 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red3.so
run base2
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
