# session 3, call b: GPU tests (new multi-rank tests first), then an interleaved A/B of
# the tile-bound load unrolling (HEAD) vs serial loads (ub0), producer warp 5, sub-block skip, 16-col panels
O=gpurun_out/${OUT:-s3b}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q > $O/multirank.log 2>&1; echo "rc=$?" >> $O/multirank.log
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; HPS_LIB=$lib timeout 600 python bench.py --leaves 888 --steps 5 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run head$rep $L/libhps_leaf.so
  run ub0_$rep $L/libhps_leaf_ub0.so
  run pw5_$rep $L/libhps_leaf_pw5.so
  run sub1_$rep $L/libhps_leaf_sub1.so
  run sp16_$rep $L/libhps_leaf_sp16.so
done
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
