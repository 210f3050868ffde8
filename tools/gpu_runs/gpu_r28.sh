TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest28.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest28.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/b28_n1.log 2>&1; echo n1=$?; tail -1 gpurun_out/b28_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['roofline']['frac'], d['gpu_launches'])"
timeout 900 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/b28_n2.log 2>&1; echo n2=$?; tail -1 gpurun_out/b28_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d.get('one_path'), d.get('host_links'))"
