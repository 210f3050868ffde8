TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/topo26.txt 2>&1; cat gpurun_out/topo26.txt | head -12
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_links tools/probe_links.cu 2>/dev/null && timeout 300 /tmp/probe_links > gpurun_out/probe_links26.txt 2>&1; echo probe=$?; grep -i "concurr\|each\|total" gpurun_out/probe_links26.txt | head
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d.get("one_path"), d.get("host_links"), d["config"]["last_step_ms_per_engine"])'
timeout 900 $TR --nproc-per-node 4 --master-port 29651 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/b26_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/b26_n4.log | python -c "$J"
