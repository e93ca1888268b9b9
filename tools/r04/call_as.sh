# session 3, call as: endgame sharing opt-in — GPU tests, smoke, default bench, determinism (15 runs)
O=gpurun_out/${OUT:-s3as}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python tools/r04/determinism.py 20 300 15 >> $O/det.jsonl 2>> $O/det.err
