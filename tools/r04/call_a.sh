# session 3 of round 2, call a: HEAD GPU tests (incl. the new multi-rank tests), smoke, per-op breakdown p16/p20, p-sweep refresh
O=gpurun_out/${OUT:-s3a}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q > $O/multirank.log 2>&1; echo "rc=$?" >> $O/multirank.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16.txt 2>&1
timeout 300 python tools/prof_breakdown.py --p 20 --leaves 296 > $O/prof20.txt 2>&1
timeout 900 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
ls -la $O
