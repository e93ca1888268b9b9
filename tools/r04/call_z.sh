# session 3, call z: W-block threshold lowered to p >= 14 — GPU tests, p = 13 / 14 A/B, p-sweep
O=gpurun_out/${OUT:-s3z}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
run() { name=$1; shift; timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
run_old() { name=$1; shift; HPS_WT_MIN_N=2048 timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
run_wt() { name=$1; shift; HPS_WT_MIN_N=0 timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p14_head_$rep --p 14 --leaves 1776 --steps 5 --warmup 3
  run_old p14_old_$rep --p 14 --leaves 1776 --steps 5 --warmup 3
  run p13_head_$rep --p 13 --leaves 2368 --steps 5 --warmup 3
  run_wt p13_wt_$rep --p 13 --leaves 2368 --steps 5 --warmup 3
done
timeout 900 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
