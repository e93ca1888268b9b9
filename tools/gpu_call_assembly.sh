# device interface assembly: GPU tests + assembly timing vs the host scatter
set -x
O=gpurun_out/c7; mkdir -p $O
timeout 600 python -m pytest tests/test_interface_assembly.py tests/test_gpu_pipeline.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 900 python tools/assembly_bench.py --N 1e6 --ps 8,12,16 > $O/assembly.jsonl 2> $O/assembly.err
timeout 600 python tools/assembly_bench.py --N 2.6e5 --ps 6,10,16 >> $O/assembly.jsonl 2>> $O/assembly.err
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
ls -la $O
