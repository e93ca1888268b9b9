# round 2: sustained A/B (power cap) of the round-2 kernel vs the round-1 GEMM settings, with power samples
O=gpurun_out/${OUT:-r2o}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run new
run old HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_old.so
run new2
run old2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_old.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks'])"; done
