# round 2: sub-block skipping with the mask frozen once a tile's sub-blocks are all active
O=gpurun_out/${OUT:-r2q}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run sub
run nosub HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nosub.so
run sub2
run nosub2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nosub.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], d['parity']['ok'])"; done
