# round 2: new defaults (warp swizzle + red epilogue): full GPU tests, A/B vs the old kernel, profile
O=gpurun_out/${OUT:-r2k}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 888 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run new
run old HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_old.so
run new2
run old2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_old.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof_p16.txt 2>&1
tail -3 $O/gpu_tests.log; grep -A3 "executed DMMA" $O/prof_p16.txt
