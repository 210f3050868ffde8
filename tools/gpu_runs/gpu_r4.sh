set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/b_n2.log 2>&1; echo n2=$?; tail -1 gpurun_out/b_n2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 3 --warmup 2 > gpurun_out/b_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/b_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --steps 3 --warmup 2 --pd 1:3 --no-cpu-baseline > gpurun_out/b_n4_1p3d.log 2>&1; echo n4_1p3d=$?; tail -1 gpurun_out/b_n4_1p3d.log
timeout 900 $TR --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 2 --warmup 1 --workload c3 --sessions-per-gpu 4 --no-cpu-baseline > gpurun_out/b_n4_c3.log 2>&1; echo n4_c3=$?; tail -1 gpurun_out/b_n4_c3.log
timeout 900 $TR --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 2 --warmup 1 --workload c2 --cap-gbps 6.25 --sessions-per-gpu 3 --no-cpu-baseline > gpurun_out/b_n4_c2cap.log 2>&1; echo n4_c2cap=$?; tail -1 gpurun_out/b_n4_c2cap.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/b_ref_n1.log 2>&1; echo ref1=$?; tail -1 gpurun_out/b_ref_n1.log
