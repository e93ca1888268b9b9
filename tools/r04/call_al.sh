# session 3, call af: tile bound loads in one pass (HEAD) vs per table (op0)
O=gpurun_out/${OUT:-s3al}; mkdir -p $O
L=paper_2503_04033_b200/_lib
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
grep -q "smoke rc=0" $O/smoke.log || exit 3
for p in 12 16 20; do timeout 600 python tools/r04/same_maps.py $L/libhps_leaf.so $L/libhps_leaf_op0.so $p 300 >> $O/same_maps.jsonl 2>> $O/same_maps.err; done
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  for v in head:libhps_leaf op0:libhps_leaf_op0; do
    n=${v%%:*}; lib=$L/${v##*:}.so
    run p16_${n}_$rep $lib --leaves 888 --steps 5 --warmup 3
    run c1_${n}_$rep $lib --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  done
done
for rep in 1 2; do
  for v in head:libhps_leaf op0:libhps_leaf_op0; do
    n=${v%%:*}; lib=$L/${v##*:}.so
    run p20_${n}_$rep $lib --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
  done
done
cat $O/same_maps.jsonl
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests_glb4.log
