TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu7.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu7.log
timeout 600 python tools/interference.py > gpurun_out/interference3.log 2>&1; echo interf=$?; tail -1 gpurun_out/interference3.log
timeout 600 python bench.py --gpus 1 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 8 --no-cpu-baseline > gpurun_out/b7_n1_c3.log 2>&1; echo c3n1=$?; tail -1 gpurun_out/b7_n1_c3.log
timeout 900 $TR --nproc-per-node 2 --master-port 29551 bench.py --gpus 2 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 8 --no-cpu-baseline --no-one-path > gpurun_out/b7_n2_c3.log 2>&1; echo c3n2=$?; tail -1 gpurun_out/b7_n2_c3.log
timeout 900 $TR --nproc-per-node 4 --master-port 29552 bench.py --gpus 4 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 8 --no-cpu-baseline --no-one-path > gpurun_out/b7_n4_c3.log 2>&1; echo c3n4=$?; tail -1 gpurun_out/b7_n4_c3.log
