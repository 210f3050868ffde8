TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["value"], d.get("model_prediction_gbps"), d.get("round_robin"), d.get("balance"), d["config"]["read_gb_per_engine"])'
timeout 900 $TR --nproc-per-node 2 --master-port 29731 bench.py --gpus 2 --steps 3 --warmup 3 --online 2 --caps 6.25,3.125 --sessions-per-gpu 4 --no-cpu-baseline > gpurun_out/b39_n2_c5.log 2>&1; echo n2_c5=$?; tail -1 gpurun_out/b39_n2_c5.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29732 bench.py --gpus 4 --steps 3 --warmup 3 --online 4 --caps 6.25,3.125,6.25,3.125 --sessions-per-gpu 4 --no-cpu-baseline > gpurun_out/b39_n4_c5.log 2>&1; echo n4_c5=$?; tail -1 gpurun_out/b39_n4_c5.log | python -c "$J"
