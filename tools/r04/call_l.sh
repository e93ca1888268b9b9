# session 3, call l: TMA producer in warp 5 (the tile's last-starting 32x32 block) after the share-count fix
O=gpurun_out/${OUT:-s3l}; mkdir -p $O
L=paper_2503_04033_b200/_lib
HPS_LIB=$L/libhps_leaf_pw5.so timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
grep -q "smoke rc=0" $O/smoke.log || exit 3
HPS_LIB=$L/libhps_leaf_pw5.so timeout 180 python bench.py --leaves 888 --steps 1 --warmup 1 --no-e2e --no-cpu --configs3-steps 0 > $O/pw5_quick.json 2> $O/pw5_quick.err; echo "quick rc=$?" >> $O/smoke.log
grep -q "quick rc=0" $O/smoke.log || exit 4
HPS_LIB=$L/libhps_leaf_pw5.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x > $O/gpu_tests_pw5.log 2>&1; echo "rc=$?" >> $O/gpu_tests_pw5.log
run() { name=$1; lib=$2; shift 2; HPS_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --configs3-steps 0 "$@" > $O/$name.json 2> $O/$name.err; }
for rep in 1 2 3; do
  run p16_head_$rep $L/libhps_leaf.so --leaves 888 --steps 5 --warmup 3
  run p16_pw5_$rep $L/libhps_leaf_pw5.so --leaves 888 --steps 5 --warmup 3
done
for rep in 1 2; do
  run p20_head_$rep $L/libhps_leaf.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
  run p20_pw5_$rep $L/libhps_leaf_pw5.so --p 20 --kappa 80 --leaves 296 --steps 2 --warmup 3
done
HPS_LIB=$L/libhps_leaf_profg.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_profg.txt 2>&1
HPS_LIB=$L/libhps_leaf_pw5profg.so timeout 300 python tools/prof_breakdown.py --p 16 --leaves 592 > $O/prof16_pw5profg.txt 2>&1
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
