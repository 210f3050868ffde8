TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 120 python tools/prof_k5.py > gpurun_out/k5.txt 2>&1; echo k5=$?; cat gpurun_out/k5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_prefill_attend -s 3 -c 1 -o gpurun_out/r01_k5_full -f python tools/prof_k5.py > gpurun_out/k5_ncu.log 2>&1; echo ncu=$?
for k1 in sm ce; do
timeout 900 $TR --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 --steps 3 --warmup 3 --prefill --k1 $k1 --no-cpu-baseline > gpurun_out/b23_n2_prefill_$k1.log 2>&1; echo n2_$k1=$?; tail -1 gpurun_out/b23_n2_prefill_$k1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; print(d['value'], d['tokens_per_s'], p['step_ms'], p['load_only_ms'], p['compute_alone_ms'], p['overlap'], d.get('one_path'))"
done
timeout 600 python bench.py --steps 3 --warmup 3 --prefill --no-cpu-baseline > gpurun_out/b23_n1_prefill.log 2>&1; echo n1=$?; tail -1 gpurun_out/b23_n1_prefill.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; print(d['value'], d['tokens_per_s'], p['step_ms'], p['load_only_ms'], p['compute_alone_ms'], p['overlap'], p['k5_tmacs'])"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest23.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest23.log
