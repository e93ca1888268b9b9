# session 3, call ar: final verification of HEAD (sharing fence): GPU tests, determinism, default bench, reference arm, configs[1], p-sweep, ncu
O=gpurun_out/${OUT:-s3ar}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --p 12 --boxes 8 --kappa 10 --field const --steps 20 --warmup 5 --configs3-steps 0 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 1200 python tools/r04/determinism.py 20 300 30 >> $O/det.jsonl 2>> $O/det.err
timeout 900 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
CL="python bench.py --steps 2 --warmup 3 --no-cpu --configs3-steps 2"
$CL > $O/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CL > $O/ncu_launch.log 2>&1
C16="python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0"
$C16 > $O/plain16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hps_leaf_kernel -s 3 -c 1 -o $O/full16 $C16 > $O/ncu_full16.log 2>&1
ls -la $O
