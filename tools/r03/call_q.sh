# L2 eviction hints on operand loads (KC 32 ring, C prefetch 2 chunks early): throughput + DRAM bytes
O=gpurun_out/${OUT:-s2q}; mkdir -p $O
L=paper_2503_04033_b200/_lib
for v in cpf2 h1 h2 h3 h3k; do
  HPS_LIB=$L/libhps_leaf_$v.so timeout 600 python bench.py --leaves 888 --steps 5 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$v.json 2> $O/$v.err
done
for v in cpf2 h1 h2 h3 h3k; do
  HPS_LIB=$L/libhps_leaf_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:hps_leaf_kernel -s 3 -c 1 --csv python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/ncu_$v.csv 2> $O/ncu_$v.err
done
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
for v in cpf2 h1 h2 h3 h3k; do echo "== $v"; grep -E 'dram__bytes|lts__t_sector_hit|gpu__time' $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}'; done
