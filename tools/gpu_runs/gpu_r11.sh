TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python tools/prof_kernels.py --k3 --reps 2 > gpurun_out/prof_k3b.log 2>&1; echo k3=$?; tail -1 gpurun_out/prof_k3b.log
timeout 900 $TR --nproc-per-node 2 --master-port 29581 bench.py --gpus 2 --steps 3 --warmup 2 --handoff --no-cpu-baseline --no-one-path > gpurun_out/b11_n2_ho.log 2>&1; echo n2ho=$?; tail -1 gpurun_out/b11_n2_ho.log
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_handoff.py -m gpu -q -x > gpurun_out/pytest11.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest11.log
