# round 2: GEMM pipeline depth sweep (k-chunk x stages), p = 16, 592 leaves (2 waves)
O=gpurun_out/${OUT:-r2c}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run kc8s4 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_kc8s4.so
run kc8s5 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_kc8s5.so
run kc8s6 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_kc8s6.so
run one_cta HPS_DEBUG=8
run base2
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
