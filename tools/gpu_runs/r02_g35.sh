# r02 call 35 (4 GPUs): the N=4 default line on the final code, and the block-major copy-engine variant
mkdir -p gpurun_out
timeout 1800 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g35_bench_n4.log 2>&1; echo n4=$?; tail -n 1 gpurun_out/g35_bench_n4.log | cut -c1-200
timeout 1200 python bench.py --gpus 4 --steps 3 --warmup 3 --no-capped --no-cpu-baseline --pool-layout block --k1 ce --k2 ce > gpurun_out/g35_bench_n4_block.log 2>&1; echo n4b=$?; tail -n 1 gpurun_out/g35_bench_n4_block.log | cut -c1-200
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "four_gpus" > gpurun_out/g35_pytest.log 2>&1; echo pytest=$?; tail -n 1 gpurun_out/g35_pytest.log
