# round 2: warp -> (row, column) block swizzle across SM sub-partitions
O=gpurun_out/${OUT:-r2j}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 888 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run wsw HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_wsw.so
run wswred HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_wswred.so
run red3 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red3.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
