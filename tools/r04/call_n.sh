# session 3, call n: line-output column chunk 16 (HEAD) vs 8 (cw8) at p = 8 / 10 / 12; GPU tests on HEAD
O=gpurun_out/${OUT:-s3n}; mkdir -p $O
L=paper_2503_04033_b200/_lib
timeout 1200 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run c1_head_$rep $L/libhps_leaf.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  run c1_cw8_$rep $L/libhps_leaf_cw8.so --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3
  run p8_head_$rep $L/libhps_leaf.so --p 8 --leaves 5920 --steps 10 --warmup 3
  run p8_cw8_$rep $L/libhps_leaf_cw8.so --p 8 --leaves 5920 --steps 10 --warmup 3
  run p10_head_$rep $L/libhps_leaf.so --p 10 --leaves 2960 --steps 10 --warmup 3
  run p10_cw8_$rep $L/libhps_leaf_cw8.so --p 10 --leaves 2960 --steps 10 --warmup 3
done
HPS_LIB=$L/libhps_leaf.so timeout 300 python tools/prof_breakdown.py --p 12 --leaves 2960 > $O/prof12_head.txt 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
