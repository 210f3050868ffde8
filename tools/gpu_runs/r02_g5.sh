# r02 call 5: staged K1/K2 parity + executor; N=1 bench sm vs staged
T="timeout 900 python -m pytest -q -p no:cacheprovider"
$T tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_prefill.py -k "staged or numa" > gpurun_out/g5_staged.log 2>&1; echo staged=$?; tail -2 gpurun_out/g5_staged.log
timeout 900 python bench.py --steps 3 --warmup 2 --k1 staged --no-cpu-baseline > gpurun_out/g5_bench_staged.log 2>&1; echo bstaged=$?; tail -1 gpurun_out/g5_bench_staged.log | cut -c1-600
timeout 900 python bench.py --steps 3 --warmup 2 --k1 staged --stage-ctas 8 --no-cpu-baseline > gpurun_out/g5_bench_staged8.log 2>&1; echo bstaged8=$?; tail -1 gpurun_out/g5_bench_staged8.log | cut -c1-300
