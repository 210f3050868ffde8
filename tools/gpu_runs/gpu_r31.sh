TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest31.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest31.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["tokens_per_s"], d.get("handoff",{}).get("gbps"), d.get("persist",{}).get("gbps"), {k: d["prefill"][k] for k in ("step_ms","load_only_ms","compute_alone_ms","overlap")}, d.get("one_path"))'
timeout 900 $TR --nproc-per-node 2 --master-port 29691 bench.py --gpus 2 --steps 3 --warmup 3 --prefill --handoff --no-cpu-baseline > gpurun_out/b31_n2_pf_ho.log 2>&1; echo n2_pf_ho=$?; tail -1 gpurun_out/b31_n2_pf_ho.log | python -c "$J"
timeout 900 $TR --nproc-per-node 2 --master-port 29692 bench.py --gpus 2 --steps 3 --warmup 3 --prefill --persist --no-cpu-baseline > gpurun_out/b31_n2_pf_p.log 2>&1; echo n2_pf_p=$?; tail -1 gpurun_out/b31_n2_pf_p.log | python -c "$J"
