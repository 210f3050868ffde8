TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d.get("one_path"), d.get("host_links",{}) and d["host_links"]["concurrent_h2d_gbps"], d["clocks"]["sm_mhz"], d["gpu_launches"])'
timeout 600 python bench.py > gpurun_out/b37_n1.log 2>&1; echo n1=$?; tail -1 gpurun_out/b37_n1.log | python -c "$J"
timeout 600 python bench.py --impl reference > gpurun_out/b37_ref1.log 2>&1; echo ref1=$?; tail -1 gpurun_out/b37_ref1.log | cut -c1-200
timeout 900 $TR --nproc-per-node 2 --master-port 29711 bench.py --gpus 2 > gpurun_out/b37_n2.log 2>&1; echo n2=$?; tail -1 gpurun_out/b37_n2.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29712 bench.py --gpus 4 > gpurun_out/b37_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/b37_n4.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29713 bench.py --gpus 4 --impl reference > gpurun_out/b37_ref4.log 2>&1; echo ref4=$?; tail -1 gpurun_out/b37_ref4.log | cut -c1-200
nvidia-smi topo -m > gpurun_out/topo37.txt 2>&1
