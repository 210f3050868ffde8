TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["value"], d.get("model_prediction_gbps"), d.get("one_path"), d.get("host_links"))'
R='import json,sys; d=json.loads(sys.stdin.read()); print("ref", d["n_gpus"], d["value"], d.get("link_model"), d["reference_wall_s_per_run"])'
timeout 900 $TR --nproc-per-node 4 --master-port 29721 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/b38_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/b38_n4.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29722 bench.py --gpus 4 --impl reference > gpurun_out/b38_ref4.log 2>&1; echo ref4=$?; tail -1 gpurun_out/b38_ref4.log | python -c "$R"
timeout 900 $TR --nproc-per-node 2 --master-port 29723 bench.py --gpus 2 --impl reference > gpurun_out/b38_ref2.log 2>&1; echo ref2=$?; tail -1 gpurun_out/b38_ref2.log | python -c "$R"
