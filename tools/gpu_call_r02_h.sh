# round 2: warp-slot utilisation of the GEMM chunks + red epilogue / 4 stages / swizzled A
O=gpurun_out/${OUT:-r2h}; mkdir -p $O
HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_profx.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof_p16.txt 2>&1
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run red3 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red3.so
run red4a0 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_red4a0.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
grep -A3 "executed DMMA" $O/prof_p16.txt
