# L2 prefetch distance sweep (diagnostic variants built by tools/build_variant.py)
O=gpurun_out/c5; mkdir -p $O
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" > $O/$name.json 2> $O/$name.err; }
L=paper_2503_04033_b200/_lib
for p in 16 20; do
  lv=592; [ $p = 20 ] && lv=296
  run base_p$p $L/libhps_leaf.so --p $p --leaves $lv
  for v in 2 4 8; do run pf${v}_p$p $L/libhps_leaf_pf$v.so --p $p --leaves $lv; done
  run base2_p$p $L/libhps_leaf.so --p $p --leaves $lv
done
