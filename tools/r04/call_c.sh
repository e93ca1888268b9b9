# session 3, call c: two kernel builds in one library (KC16x3 / KC32x2 by p): GPU tests, A/B per p, p-sweep
O=gpurun_out/${OUT:-s3c}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
B="timeout 600 python bench.py --no-e2e --no-cpu --configs3-steps 0"
for rep in 1 2; do
  for kc in 16 32; do
    HPS_KC_VARIANT=$kc $B --p 12 --boxes 8 --kappa 10 --field const --steps 10 --warmup 3 > $O/c1_kc${kc}_$rep.json 2> $O/c1_kc${kc}_$rep.err
    HPS_KC_VARIANT=$kc $B --p 14 --leaves 1776 --steps 5 --warmup 3 > $O/p14_kc${kc}_$rep.json 2> $O/p14_kc${kc}_$rep.err
    HPS_KC_VARIANT=$kc $B --p 16 --leaves 888 --steps 5 --warmup 3 > $O/p16_kc${kc}_$rep.json 2> $O/p16_kc${kc}_$rep.err
  done
done
timeout 900 python tools/p_sweep.py > $O/p_sweep.jsonl 2> $O/p_sweep.err
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
