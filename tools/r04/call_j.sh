# session 3, call j: next-tile A prefetch for the latency-bound narrow / tall GEMMs (HPS_PF_NEXT 2 / 4) A/B + breakdowns
O=gpurun_out/${OUT:-s3j}; mkdir -p $O
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_pfn4_$rep $L/libhps_leaf_pfn4.so --leaves 888 --steps 5 --warmup 3
  run p16_pfn2_$rep $L/libhps_leaf_pfn2.so --leaves 888 --steps 5 --warmup 3
done
HPS_LIB=$L/libhps_leaf.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_head.txt 2>&1
HPS_LIB=$L/libhps_leaf_pfn4.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_pfn4.txt 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
