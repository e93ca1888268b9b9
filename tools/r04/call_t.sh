# session 3, call t: deferred column bookkeeping — more interleaved reps at p = 8 / 12
O=gpurun_out/${OUT:-s3t}; mkdir -p $O
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3 4; do
  run c1_head_$rep $L/libhps_leaf.so --p 12 --boxes 8 --kappa 10 --field const --steps 20 --warmup 3
  run c1_defer0_$rep $L/libhps_leaf_defer0.so --p 12 --boxes 8 --kappa 10 --field const --steps 20 --warmup 3
  run p8_head_$rep $L/libhps_leaf.so --p 8 --leaves 5920 --steps 20 --warmup 3
  run p8_defer0_$rep $L/libhps_leaf_defer0.so --p 8 --leaves 5920 --steps 20 --warmup 3
done
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
