# r02 call 28 (2 GPUs): the final code -- the full suite on 2 GPUs, the suite as a 1-GPU box sees it, smoke
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g28_pytest_2gpu.log 2>&1; echo two=$?; tail -n 2 gpurun_out/g28_pytest_2gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g28_pytest_1gpu.log 2>&1; echo one=$?; tail -n 2 gpurun_out/g28_pytest_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g28_smoke.log
