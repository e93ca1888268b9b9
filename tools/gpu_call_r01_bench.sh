# round-1 bench lines with the per-warp work model (run under gpurun from the repo root)
set -x
O=gpurun_out/c3; mkdir -p $O
timeout 500 python bench.py > $O/bench_p16.json 2> $O/bench_p16.err
timeout 400 python bench.py --p 20 --leaves 512 --kappa 80 --steps 3 --warmup 3 > $O/bench_p20.json 2> $O/bench_p20.err
timeout 300 python bench.py --p 12 --boxes 8 --kappa 10 --field const > $O/bench_p12.json 2> $O/bench_p12.err
timeout 600 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
ls -la $O
