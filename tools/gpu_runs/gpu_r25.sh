TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("e2e",{}).get("value"), d["roofline"]["frac"], d.get("one_path"), d.get("tier",{}).get("io_wait_ms_max_step"), d.get("prefill",{}).get("overlap"), d["clocks"])'
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest25.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest25.log
timeout 600 python bench.py > gpurun_out/b25_n1.log 2>&1; echo n1=$?; tail -1 gpurun_out/b25_n1.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29651 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/b25_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/b25_n4.log | python -c "$J"
for t in 8 16; do
timeout 900 python bench.py --steps 3 --warmup 3 --tier /tmp/dp_tier.bin --io-threads $t --no-cpu-baseline > gpurun_out/b25_n1_tier$t.log 2>&1; echo n1_tier$t=$?; tail -1 gpurun_out/b25_n1_tier$t.log | python -c "$J"
done
timeout 900 $TR --nproc-per-node 4 --master-port 29652 bench.py --gpus 4 --steps 3 --warmup 3 --prefill --no-cpu-baseline > gpurun_out/b25_n4_prefill.log 2>&1; echo n4p=$?; tail -1 gpurun_out/b25_n4_prefill.log | python -c "$J"
