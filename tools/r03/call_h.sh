O=gpurun_out/${OUT:-s2h}; mkdir -p $O
for v in notma notmaidle apad0 bpad0; do for c in 1 2; do timeout 300 ./tools/gemm/gemm_bench_$v $c > $O/gemm_${v}_$c.txt 2>&1; done; done
