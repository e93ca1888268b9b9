# round 2: driver-style measurements on the current kernel
O=gpurun_out/${OUT:-r2m}; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --p 12 --boxes 8 --kappa 10 --field const --configs3-steps 0 --steps 5 > $O/bench_c1_p12.json 2> $O/bench_c1_p12.err
timeout 900 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
ls -la $O
