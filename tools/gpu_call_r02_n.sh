# round 2: panel block width from the compacted candidate count — tests and A/B at p=16 / p=20
O=gpurun_out/${OUT:-r2n}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 888 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run cwb
run nocwb HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nocwb.so
run20() { name=$1; shift; env "$@" timeout 300 python bench.py --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run20 cwb20
run20 nocwb20 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nocwb.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['parity']['ok'])"; done
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 20 --leaves 296 > $O/prof_p20.txt 2>&1
tail -3 $O/gpu_tests.log; head -25 $O/prof_p20.txt
