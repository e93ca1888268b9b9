# session 3, call h: non-volatile DMMA asm (HPS_DMMA_NV=1: the compiler may schedule around the DMMAs) A/B
O=gpurun_out/${OUT:-s3h}; mkdir -p $O
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_nv1_$rep $L/libhps_leaf_nv1.so --leaves 888 --steps 5 --warmup 3
done
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
