# session 3, call ac: boundary rows per W block (HPS_RW_ROWS runtime override) at p = 16 / 20 / 14
O=gpurun_out/${OUT:-s3ac}; mkdir -p $O
run() { name=$1; rw=$2; shift 2; HPS_RW_ROWS=$rw timeout 400 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  for rw in 256 512 1184; do run p16_rw${rw}_$rep $rw --leaves 888 --steps 5 --warmup 3; done
  for rw in 256 512 1024; do run p20_rw${rw}_$rep $rw --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3; done
  for rw in 256 448 896; do run p14_rw${rw}_$rep $rw --p 14 --leaves 1776 --steps 5 --warmup 3; done
done
