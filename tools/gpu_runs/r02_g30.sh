# r02 call 30 (1 GPU): every kernel once on small stream-ordered cases (incl. the copy-engine K3 and the staged K4)
mkdir -p gpurun_out
timeout 300 python tools/sanitize/kernels_small.py > gpurun_out/g30_kernels_small.log 2>&1; echo small=$?; tail -n 3 gpurun_out/g30_kernels_small.log
