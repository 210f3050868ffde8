# r02 call 23 (2 GPUs): new edge-case tests (K3 copy path > 48 jobs, staged K4 with interleaved requests),
# the suite as the driver's 1-GPU box sees it, the launch list of K3 / K4 alone (side kernel, persist gather)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "many_jobs or two_requests" > gpurun_out/g23_pytest_new.log 2>&1; echo new=$?; tail -n 2 gpurun_out/g23_pytest_new.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g23_pytest_1gpu.log 2>&1; echo one=$?; tail -n 2 gpurun_out/g23_pytest_1gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g23_k3k4_launches.csv python tools/prof_kernels.py --k3 --k4 --reps 1 > gpurun_out/g23_ncu.log 2>&1; echo ncu=$?
