# r02 call 17 (2 GPUs): K3 copy path without the helper stream (g16: 2 PEs on one GPU deadlocked),
# the one-hardware-queue test, K3/K4 alone (K4 staged with session-contiguous Full Blocks),
# online capacity with the first-token TTFT (SLO 1 s)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g17_pytest.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/g17_pytest.log
timeout 400 python tools/prof_kernels.py --k3 --k4 --peer > gpurun_out/g17_k3k4.json 2> gpurun_out/g17_k3k4.err; echo prof=$?; cat gpurun_out/g17_k3k4.json
timeout 1500 python tools/online_capacity.py --pd 1:1 --prefill --handoff --slo 1.0 --bisect 2 > gpurun_out/g17_online_handoff.json 2> gpurun_out/g17_online_handoff.err; echo onlineh=$?; tail -n 2 gpurun_out/g17_online_handoff.err
