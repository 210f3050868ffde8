TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest14.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest14.log
timeout 300 python tools/prof_kernels.py --k2 --k3 --k3-ctas 0,296 --reps 2 > gpurun_out/prof_k3d.log 2>&1; echo k3=$?; tail -1 gpurun_out/prof_k3d.log
timeout 900 $TR --nproc-per-node 2 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 2 --handoff --no-cpu-baseline --no-one-path > gpurun_out/b14_n2_ho.log 2>&1; echo n2ho=$?; tail -1 gpurun_out/b14_n2_ho.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['handoff']['gbps'], d['config']['last_step_ms_per_engine'])"
