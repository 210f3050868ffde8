TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 ./tools/probe_ce > gpurun_out/probe_ce.txt 2>&1; echo probe_ce=$?; cat gpurun_out/probe_ce.txt
timeout 300 python tools/prof_kernels.py --k2 --shape qwen --jobs 16 --blocks 64 > gpurun_out/prof_qwen.log 2>&1; echo qwen=$?; tail -1 gpurun_out/prof_qwen.log
timeout 600 python tools/interference.py > gpurun_out/interference2.log 2>&1; echo interf=$?; tail -1 gpurun_out/interference2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29541 bench.py --gpus 4 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 8 --no-cpu-baseline > gpurun_out/b6_n4_c3.log 2>&1; echo c3=$?; tail -1 gpurun_out/b6_n4_c3.log
timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q > gpurun_out/pytest_engine6.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_engine6.log
