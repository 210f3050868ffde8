TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest15.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest15.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke15.log
timeout 600 python bench.py > gpurun_out/b15_default.log 2>&1; echo default=$?; tail -1 gpurun_out/b15_default.log
timeout 600 python bench.py --impl reference > gpurun_out/b15_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/b15_ref.log
timeout 900 $TR --nproc-per-node 4 --master-port 29621 bench.py --gpus 4 --steps 3 --warmup 2 --handoff --no-cpu-baseline > gpurun_out/b15_n4_ho.log 2>&1; echo n4ho=$?; tail -1 gpurun_out/b15_n4_ho.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['handoff']['gbps'], d.get('one_path'), d['config']['last_step_ms_per_engine'])"
timeout 900 $TR --nproc-per-node 4 --master-port 29622 bench.py --gpus 4 --impl reference > gpurun_out/b15_ref4.log 2>&1; echo ref4=$?; tail -1 gpurun_out/b15_ref4.log
