# call b: idle-warp DMMA probe; C-prefetch timing / serpentine-k variants: throughput + DRAM bytes
O=gpurun_out/${OUT:-s2b}; mkdir -p $O
for v in idle_hi idle_odd; do timeout 300 ./tools/gemm/gemm_bench_$v 2 > $O/gemm_${v}_2.txt 2>&1; timeout 300 ./tools/gemm/gemm_bench_$v 1 > $O/gemm_${v}_1.txt 2>&1; done
L=paper_2503_04033_b200/_lib
run() { name=$1; lib=$2; HPS_LIB=$lib timeout 600 python bench.py --leaves 888 --steps 5 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/$name.json 2> $O/$name.err; }
for v in base cpf2 cpf4 krev krevcpf4; do
  if [ $v = base ]; then lib=$L/libhps_leaf.so; else lib=$L/libhps_leaf_$v.so; fi
  run $v $lib
done
for v in base cpf4 krev krevcpf4; do
  if [ $v = base ]; then lib=$L/libhps_leaf.so; else lib=$L/libhps_leaf_$v.so; fi
  HPS_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:hps_leaf_kernel -s 3 -c 1 --csv python bench.py --leaves 296 --steps 1 --warmup 3 --no-e2e --no-cpu --configs3-steps 0 > $O/ncu_$v.csv 2> $O/ncu_$v.err
done
for f in $O/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), d['parity']['ok'])"; done
