# session 3, call x: HEAD sanity after the last bench.py change — GPU tests, smoke, a short bench line
O=gpurun_out/${OUT:-s3x}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 5 --configs3-steps 1 > $O/bench_short.json 2> $O/bench_short.err
