# r02 call 2: debug the two same-GPU failures (first dual test; tight persistence)
T="timeout 300 python -m pytest -q -p no:cacheprovider -x"
$T "tests/test_gpu_handoff.py::test_de_path_dual_then_missmerge" -k "same_gpu and 330" > gpurun_out/g2_a_default.log 2>&1; echo a_default=$?
CUDA_MODULE_LOADING=EAGER $T "tests/test_gpu_handoff.py::test_de_path_dual_then_missmerge" -k "same_gpu and 330" > gpurun_out/g2_a_eager.log 2>&1; echo a_eager=$?
$T tests/test_gpu_engine.py::test_handoff_with_persistence -k "same_gpu and True" > gpurun_out/g2_b_default.log 2>&1; echo b_default=$?
CUDA_MODULE_LOADING=EAGER $T tests/test_gpu_engine.py::test_handoff_with_persistence -k "same_gpu and True" > gpurun_out/g2_b_eager.log 2>&1; echo b_eager=$?
CUDA_DEVICE_MAX_CONNECTIONS=8 $T tests/test_gpu_engine.py::test_handoff_with_persistence -k "same_gpu and True" > gpurun_out/g2_b_conn8.log 2>&1; echo b_conn8=$?
tail -3 gpurun_out/g2_*.log
