# session 3, call e: operand L2 prefetch ahead of the 2-stage ring (HPS_PF 1/2) A/B; ncu full capture of HEAD at p=16
O=gpurun_out/${OUT:-s3e}; mkdir -p $O
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_pf1_$rep $L/libhps_leaf_pf1.so --leaves 888 --steps 5 --warmup 3
  run p16_pf2_$rep $L/libhps_leaf_pf2.so --leaves 888 --steps 5 --warmup 3
done
C16="python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0"
$C16 > $O/plain16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hps_leaf_kernel -s 3 -c 1 -o $O/full16 $C16 > $O/ncu_full16.log 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
ls -la $O
