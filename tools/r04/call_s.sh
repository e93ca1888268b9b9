# session 3, call o: pivot search with integer keys + warp reductions (HEAD) vs FP64 compares (defer0)
O=gpurun_out/${OUT:-s3s}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for p in 8 12 16; do timeout 300 python tools/r04/same_maps.py $L/libhps_leaf.so $L/libhps_leaf_defer0.so $p 600 >> $O/same_maps.jsonl 2>> $O/same_maps.err; done
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run c1_head_$rep $L/libhps_leaf.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  run c1_defer0_$rep $L/libhps_leaf_defer0.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  run p8_head_$rep $L/libhps_leaf.so --p 8 --leaves 5920 --steps 10 --warmup 3
  run p8_defer0_$rep $L/libhps_leaf_defer0.so --p 8 --leaves 5920 --steps 10 --warmup 3
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_defer0_$rep $L/libhps_leaf_defer0.so --leaves 888 --steps 5 --warmup 3
done
HPS_LIB=$L/libhps_leaf.so timeout 300 python tools/prof_breakdown.py --p 12 --leaves 2960 > $O/prof12_head.txt 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
cat $O/same_maps.jsonl
HPS_LIB=$L/libhps_leaf_profpiv.so timeout 300 python tools/prof_breakdown.py --p 12 --leaves 2960 > $O/prof12_piv.txt 2>&1
