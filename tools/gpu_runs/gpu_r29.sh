TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x -k "copy_engine" > gpurun_out/pytest29.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest29.log
timeout 300 python tools/de_interference.py > gpurun_out/de_int.json 2> gpurun_out/de_int.err; echo de_int=$?; cat gpurun_out/de_int.json; tail -2 gpurun_out/de_int.err
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("one_path"), d.get("host_links",{}).get("value_frac") if d.get("host_links") else None, d["config"]["last_step_ms_per_engine"])'
timeout 900 $TR --nproc-per-node 2 --master-port 29681 bench.py --gpus 2 --k2 ce --no-cpu-baseline > gpurun_out/b29_n2_k2ce.log 2>&1; echo n2_k2ce=$?; tail -1 gpurun_out/b29_n2_k2ce.log | python -c "$J"
timeout 900 $TR --nproc-per-node 2 --master-port 29682 bench.py --gpus 2 --k2 ce --prefill --no-cpu-baseline > gpurun_out/b29_n2_k2ce_prefill.log 2>&1; echo n2_k2ce_pf=$?; tail -1 gpurun_out/b29_n2_k2ce_prefill.log | python -c "$J"
