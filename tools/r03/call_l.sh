O=gpurun_out/${OUT:-s2l}; mkdir -p $O
for v in base rot rotidle rots4 rottrace; do for c in 1 2; do timeout 300 ./tools/gemm/gemm_bench_$v $c > $O/gemm_${v}_$c.txt 2>&1; done; done
