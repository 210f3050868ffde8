TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu5.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu5.log
timeout 600 python tools/prof_kernels.py --k2 --ctas 0,148,64,32,16,8,4,2 > gpurun_out/ctas_sweep.log 2>&1; echo ctas=$?; tail -1 gpurun_out/ctas_sweep.log
timeout 600 python tools/interference.py > gpurun_out/interference.log 2>&1; echo interf=$?; tail -1 gpurun_out/interference.log
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 2 > gpurun_out/b5_n1.log 2>&1; echo n1=$?; tail -1 gpurun_out/b5_n1.log
timeout 900 $TR --nproc-per-node 4 --master-port 29531 bench.py --gpus 4 --steps 2 --warmup 1 --workload c2 --cap-gbps 6.25 --sessions-per-gpu 3 --no-cpu-baseline > gpurun_out/b5_n4_c2cap.log 2>&1; echo c2cap=$?; tail -1 gpurun_out/b5_n4_c2cap.log
timeout 900 $TR --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 --steps 1 --warmup 1 --online 4 --caps 6.25,3.125,6.25,3.125 --sessions-per-gpu 2 --no-cpu-baseline > gpurun_out/b5_n4_c5.log 2>&1; echo c5=$?; tail -1 gpurun_out/b5_n4_c5.log
timeout 900 $TR --nproc-per-node 4 --master-port 29533 bench.py --gpus 4 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 8 --no-cpu-baseline > gpurun_out/b5_n4_c3.log 2>&1; echo c3=$?; tail -1 gpurun_out/b5_n4_c3.log
