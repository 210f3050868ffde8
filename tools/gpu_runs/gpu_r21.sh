TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/pytest21_prefill.log 2>&1; echo pytest_prefill=$?; tail -3 gpurun_out/pytest21_prefill.log
for k1 in sm ce; do
timeout 600 python bench.py --steps 3 --warmup 3 --prefill --k1 $k1 --no-cpu-baseline > gpurun_out/b21_n1_prefill_$k1.log 2>&1; echo n1_$k1=$?; tail -1 gpurun_out/b21_n1_prefill_$k1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; print(d['value'], d['tokens_per_s'], p['step_ms'], p['load_only_ms'], p['compute_alone_ms'], p['overlap'], p['k5_tmacs'])"
done
timeout 900 $TR --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 --steps 3 --warmup 3 --prefill --no-cpu-baseline > gpurun_out/b21_n2_prefill.log 2>&1; echo n2=$?; tail -1 gpurun_out/b21_n2_prefill.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; print(d['value'], d['tokens_per_s'], p['step_ms'], p['load_only_ms'], p['compute_alone_ms'], p['overlap'], d.get('one_path'))"
