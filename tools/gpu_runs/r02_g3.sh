# r02 call 3: same-GPU DE path after the stream-creation fix; flakiness of the executor tests
T="timeout 600 python -m pytest -q -p no:cacheprovider"
$T tests/test_gpu_handoff.py tests/test_gpu_kernels.py -k "same_gpu or numa" > gpurun_out/g3_kern.log 2>&1; echo kern=$?; tail -2 gpurun_out/g3_kern.log
for i in 1 2 3 4; do
  $T tests/test_gpu_engine.py tests/test_gpu_prefill.py -k "same_gpu or one_gpu" > gpurun_out/g3_eng_$i.log 2>&1; echo eng$i=$?; tail -1 gpurun_out/g3_eng_$i.log
done
