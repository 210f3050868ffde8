TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["value"], d.get("model_prediction_gbps"), d.get("one_path"), d.get("host_links"), d["plan_s"], d["config"]["last_step_ms_per_engine"])'
timeout 1500 $TR --nproc-per-node 8 --master-port 29741 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b40_n8_on4.log 2>&1; echo n8=$?; tail -1 gpurun_out/b40_n8_on4.log | python -c "$J"
timeout 900 $TR --nproc-per-node 8 --master-port 29742 bench.py --gpus 8 --steps 3 --warmup 3 --impl reference > gpurun_out/b40_ref8.log 2>&1; echo ref8=$?; tail -1 gpurun_out/b40_ref8.log | cut -c1-300
