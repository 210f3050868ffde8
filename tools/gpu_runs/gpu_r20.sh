TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest20_prefill.log 2>&1; echo pytest_prefill=$?; tail -3 gpurun_out/pytest20_prefill.log
timeout 600 python bench.py --steps 3 --warmup 3 --prefill --no-cpu-baseline > gpurun_out/b20_n1_prefill.log 2>&1; echo n1=$?; tail -1 gpurun_out/b20_n1_prefill.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['tokens_per_s'], d['prefill'])"
timeout 900 $TR --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 --steps 3 --warmup 3 --prefill --no-cpu-baseline > gpurun_out/b20_n2_prefill.log 2>&1; echo n2=$?; tail -1 gpurun_out/b20_n2_prefill.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['tokens_per_s'], d['prefill'], d.get('one_path'))"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest20.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest20.log
