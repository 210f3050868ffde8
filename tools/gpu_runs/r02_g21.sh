# r02 call 21 (2 GPUs): the final code's full 2-GPU suite (live persistence + PersistWrite), the default N=2 line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g21_pytest.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/g21_pytest.log
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g21_bench_n2.log 2>&1; echo n2=$?; tail -n 1 gpurun_out/g21_bench_n2.log | cut -c1-200
