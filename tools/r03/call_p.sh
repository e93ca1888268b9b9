# KC=32 / 2-stage ring: GPU tests, then 888-leaf bench vs the round-2 ring (KC 16 x 3), and C prefetch 2 chunks early
O=gpurun_out/${OUT:-s2p}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; HPS_LIB=$lib timeout 600 python bench.py --leaves 888 --steps 5 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
run new $L/libhps_leaf.so
run old16 $L/libhps_leaf_old16.so
run cpf2 $L/libhps_leaf_cpf2.so
run new2 $L/libhps_leaf.so
run old16b $L/libhps_leaf_old16.so
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
