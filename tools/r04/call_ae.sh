# session 3, call ae: warp producer (tile claims / k bounds over 32 lanes, HPS_WARP_PRODUCER=1) vs thread producer
O=gpurun_out/${OUT:-s3ae}; mkdir -p $O
L=paper_2503_04033_b200/_lib
HPS_LIB=$L/libhps_leaf_wp1.so timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
grep -q "smoke rc=0" $O/smoke.log || exit 3
for p in 12 16 20; do timeout 600 python tools/r04/same_maps.py $L/libhps_leaf_wp1.so $L/libhps_leaf.so $p 300 >> $O/same_maps.jsonl 2>> $O/same_maps.err; done
HPS_LIB=$L/libhps_leaf_wp1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x > $O/gpu_tests_wp1.log 2>&1; echo "rc=$?" >> $O/gpu_tests_wp1.log
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_wp1_$rep $L/libhps_leaf_wp1.so --leaves 888 --steps 5 --warmup 3
  run c1_head_$rep $L/libhps_leaf.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  run c1_wp1_$rep $L/libhps_leaf_wp1.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
done
for rep in 1 2; do
  run p20_head_$rep $L/libhps_leaf.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
  run p20_wp1_$rep $L/libhps_leaf_wp1.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
done
cat $O/same_maps.jsonl
