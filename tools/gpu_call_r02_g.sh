# round 2: red.global.add epilogue (no smem ring) with 3 / 4 stages: speed and exactness
O=gpurun_out/${OUT:-r2g}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run red3 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red3.so
run red4 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red4.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -x -q > $O/tests_red4.log 2>&1; tail -3 $O/tests_red4.log
