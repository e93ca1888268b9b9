# KC 32 / 2-stage ring, C prefetch 2 chunks early, B evict_first: GPU tests, default bench, reference arm, ncu (launch list + full p=16/p=20)
O=gpurun_out/${OUT:-s2r}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
C16="python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0"
C20="python bench.py --p 20 --kappa 80 --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0"
CL="python bench.py --steps 2 --warmup 3 --no-cpu --configs3-steps 2"
$CL > $O/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CL > $O/ncu_launch.log 2>&1
$C16 > $O/plain16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hps_leaf_kernel -s 3 -c 1 -o $O/full16 $C16 > $O/ncu_full16.log 2>&1
$C20 > $O/plain20.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hps_leaf_kernel -s 3 -c 1 -o $O/full20 $C20 > $O/ncu_full20.log 2>&1
ls -la $O
