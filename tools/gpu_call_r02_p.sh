# round 2: 8x8 sub-block DMMA skipping — tests, executed work, sustained A/B at the power cap
O=gpurun_out/${OUT:-r2p}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
tail -2 $O/gpu_tests.log
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof_p16.txt 2>&1
grep -A4 "executed DMMA" $O/prof_p16.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run sub
run nosub HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nosub.so
run sub2
run nosub2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_nosub.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], d['parity']['ok'])"; done
