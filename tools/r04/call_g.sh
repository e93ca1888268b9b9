# session 3, call g: sliced chunk production (every warp issues its slice; HPS_SLICE=1) — parity tests on the
# variant library, then interleaved A/B vs HEAD at p=16 and p=20
O=gpurun_out/${OUT:-s3g}; mkdir -p $O
L=paper_2503_04033_b200/_lib
HPS_LIB=$L/libhps_leaf_slice1.so timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
grep -q "smoke rc=0" $O/smoke.log || exit 3
HPS_LIB=$L/libhps_leaf_slice1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x > $O/gpu_tests_slice.log 2>&1; echo "rc=$?" >> $O/gpu_tests_slice.log
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_slice_$rep $L/libhps_leaf_slice1.so --leaves 888 --steps 5 --warmup 3
  run p20_head_$rep $L/libhps_leaf.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
  run p20_slice_$rep $L/libhps_leaf_slice1.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
done
HPS_LIB=$L/libhps_leaf_slice1.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_slice.txt 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
