# r02 call 34 (2 GPUs): final regression on the final code -- full suite (2 GPUs and the 1-GPU view), smoke
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g34_pytest_2gpu.log 2>&1; echo two=$?; tail -n 2 gpurun_out/g34_pytest_2gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g34_pytest_1gpu.log 2>&1; echo one=$?; tail -n 2 gpurun_out/g34_pytest_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g34_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g34_smoke.log | cut -c1-120
