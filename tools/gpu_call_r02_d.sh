# round 2: epilogue ring / A-box swizzle / W-block size variants; build() leaf-stage throughput
O=gpurun_out/${OUT:-r2d}; mkdir -p $O
run() { name=$1; shift; env "$@" timeout 300 python bench.py --leaves 592 --steps 3 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run base
run epi2 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_epi2.so
run apad0 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_apad0.so
run rw512 HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_rw512.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['parity']['ok'])"; done
timeout 1500 python tools/build_bench.py --boxes 16 --p 16 --flushes 592,1184,2048,4096 > $O/build_bench.jsonl 2> $O/build_bench.err
cat $O/build_bench.jsonl
