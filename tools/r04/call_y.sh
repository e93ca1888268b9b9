# session 3, call y: W-block Schur complement threshold — forced on (HPS_WT_MIN_N=0) vs default at p = 10 / 12 / 14
O=gpurun_out/${OUT:-s3y}; mkdir -p $O
run_wt() { name=$1; shift; HPS_WT_MIN_N=0 timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
run() { name=$1; shift; timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run c1_def_$rep --p 12 --boxes 8 --kappa 10 --field const --steps 20 --warmup 3
  run_wt c1_wt_$rep --p 12 --boxes 8 --kappa 10 --field const --steps 20 --warmup 3
  run p14_def_$rep --p 14 --leaves 1776 --steps 5 --warmup 3
  run_wt p14_wt_$rep --p 14 --leaves 1776 --steps 5 --warmup 3
  run p10_def_$rep --p 10 --leaves 2960 --steps 20 --warmup 3
  run_wt p10_wt_$rep --p 10 --leaves 2960 --steps 20 --warmup 3
done
