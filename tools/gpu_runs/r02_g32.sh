# r02 call 32 (2 GPUs): regression check after the pool-stride change -- the full suite on 2 GPUs and as a
# 1-GPU box sees it, smoke, the default N=1 line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g32_pytest_2gpu.log 2>&1; echo two=$?; tail -n 2 gpurun_out/g32_pytest_2gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g32_pytest_1gpu.log 2>&1; echo one=$?; tail -n 2 gpurun_out/g32_pytest_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g32_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g32_smoke.log | cut -c1-120
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g32_bench_n1.log 2>&1; echo n1=$?; tail -n 1 gpurun_out/g32_bench_n1.log | cut -c1-200
