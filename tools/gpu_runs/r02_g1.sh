# r02 call 1: 1-GPU DE read path (same-device peer views) — GPU tests + smoke
nvidia-smi -L > gpurun_out/g1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/g1_smoke.log
