# session 3, call v: energy per leaf of epilogue / L2-hint variants (power median during the timed region)
O=gpurun_out/${OUT:-s3v}; mkdir -p $O
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 10 --warmup 3
  run p16_epi0_$rep $L/libhps_leaf_epi0.so --leaves 888 --steps 10 --warmup 3
  run p16_h3_$rep $L/libhps_leaf_h3.so --leaves 888 --steps 10 --warmup 3
done
