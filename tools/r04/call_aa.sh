# session 3, call aa: recursive-split knobs (HPS_SPLIT_PCT, HPS_SPLIT_ALIGN; runtime env) at p = 16 and 12
O=gpurun_out/${OUT:-s3aa}; mkdir -p $O
run() { name=$1; shift; timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  for v in "50 128" "40 128" "60 128" "50 64" "50 256"; do
    set -- $v
    HPS_SPLIT_PCT=$1 HPS_SPLIT_ALIGN=$2 run p16_s$1_a$2_$rep --leaves 888 --steps 5 --warmup 3
    HPS_SPLIT_PCT=$1 HPS_SPLIT_ALIGN=$2 run c1_s$1_a$2_$rep --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  done
done
