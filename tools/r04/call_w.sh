# session 3, call w: W-block rows zeroed by bulk stores (HEAD) vs LSU stores (wbz0)
O=gpurun_out/${OUT:-s3w}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for p in 16 20; do timeout 600 python tools/r04/same_maps.py $L/libhps_leaf.so $L/libhps_leaf_wbz0.so $p 300 >> $O/same_maps.jsonl 2>> $O/same_maps.err; done
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 10 --warmup 3
  run p16_wbz0_$rep $L/libhps_leaf_wbz0.so --leaves 888 --steps 10 --warmup 3
done
for rep in 1 2; do
  run p20_head_$rep $L/libhps_leaf.so --p 20 --kappa 80 --leaves 296 --steps 3 --warmup 3
  run p20_wbz0_$rep $L/libhps_leaf_wbz0.so --p 20 --kappa 80 --leaves 296 --steps 3 --warmup 3
done
cat $O/same_maps.jsonl
