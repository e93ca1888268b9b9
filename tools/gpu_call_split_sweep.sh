O=gpurun_out/c4; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 200 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/$name.json 2> $O/$name.err; }
run base
run a64 HPS_SPLIT_ALIGN=64
run a256 HPS_SPLIT_ALIGN=256
run pct40 HPS_SPLIT_PCT=40
run pct60 HPS_SPLIT_PCT=60
run pct33 HPS_SPLIT_PCT=33
run base2
HPS_DEBUG=128 timeout 200 python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/hist.json 2> $O/hist.err
