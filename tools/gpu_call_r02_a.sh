# round 2, first call: new bench-order parity tests, the reworked bench, reference arm
set -x
O=gpurun_out/${OUT:-r2a}; mkdir -p $O
nproc > $O/nproc.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> $O/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --configs3-steps 3 > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 --ref-seconds 30 > $O/bench_reference.json 2> $O/bench_reference.err
ls -la $O
