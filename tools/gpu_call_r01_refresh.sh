set -x
O=gpurun_out/c2; mkdir -p $O
timeout 400 python bench.py --p 20 --leaves 512 --kappa 80 --steps 3 --warmup 3 > $O/bench_p20.json 2> $O/bench_p20.err
timeout 300 python bench.py --p 12 --boxes 8 --kappa 10 --field const > $O/bench_p12.json 2> $O/bench_p12.err
timeout 200 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof_p16.txt 2>&1
for v in rw128 rw512; do HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_$v.so timeout 200 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/sw_$v.json 2>&1; done
for sp in 16 24; do HPS_SMALL_PANEL=$sp timeout 200 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/sw_sp$sp.json 2>&1; done
timeout 200 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/sw_base.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hps_leaf_kernel -s 3 -c 1 -o $O/full python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
ls -la $O
