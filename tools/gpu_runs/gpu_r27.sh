TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("model_prediction_gbps"), d.get("one_path"), d.get("host_links",{}).get("concurrent_h2d_gbps") if d.get("host_links") else None)'
for cap in 3.125 6.25 12.5 25; do
timeout 1200 $TR --nproc-per-node 4 --master-port 29661 bench.py --gpus 4 --steps 3 --warmup 3 --workload c2 --sessions-per-gpu 6 --cap-gbps $cap --no-cpu-baseline > gpurun_out/b27_n4_c2_cap$cap.log 2>&1; echo c2_cap$cap=$?; tail -1 gpurun_out/b27_n4_c2_cap$cap.log | python -c "$J"
done
timeout 1200 $TR --nproc-per-node 4 --master-port 29662 bench.py --gpus 4 --steps 3 --warmup 3 --workload c3 --sessions-per-gpu 8 --pd 1:3 --no-cpu-baseline > gpurun_out/b27_n4_c3_1p3d.log 2>&1; echo c3_1p3d=$?; tail -1 gpurun_out/b27_n4_c3_1p3d.log | python -c "$J"
timeout 1200 $TR --nproc-per-node 4 --master-port 29663 bench.py --gpus 4 --steps 3 --warmup 3 --workload c3 --sessions-per-gpu 8 --pd 3:1 --no-cpu-baseline > gpurun_out/b27_n4_c3_3p1d.log 2>&1; echo c3_3p1d=$?; tail -1 gpurun_out/b27_n4_c3_3p1d.log | python -c "$J"
