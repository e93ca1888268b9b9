set -x
O=gpurun_out/c10; mkdir -p $O
timeout 600 python -m pytest tests/test_interface_assembly.py tests/test_gpu_pipeline.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python tools/scatter_bench.py --p 16 --g 6 > $O/scatter_p16.json 2> $O/scatter_p16.err
timeout 300 python tools/scatter_bench.py --p 8 --g 12 > $O/scatter_p8.json 2> $O/scatter_p8.err
timeout 300 python tools/scatter_bench.py --p 12 --g 8 > $O/scatter_p12.json 2> $O/scatter_p12.err
timeout 900 python tools/assembly_bench.py --N 1e6 --ps 8,12,16 > $O/assembly.jsonl 2> $O/assembly.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hps_interface_scatter -s 3 -c 1 -o $O/scatter_full python tools/scatter_bench.py --p 16 --g 6 --iters 1 > $O/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:hps_interface_scatter -s 3 -c 1 -o $O/scatter_full_p8 python tools/scatter_bench.py --p 8 --g 12 --iters 1 > $O/ncu8.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
ls -la $O
