TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest33.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest33.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["tokens_per_s"], d.get("handoff",{}).get("gbps"), d.get("persist",{}).get("gbps"), {k: d["prefill"][k] for k in ("step_ms","load_only_ms","compute_alone_ms","overlap")}, d.get("one_path"), d.get("host_links",{}).get("concurrent_h2d_gbps"))'
timeout 900 $TR --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 --steps 3 --warmup 3 --prefill --persist --no-cpu-baseline > gpurun_out/b33_n4_pf_p.log 2>&1; echo n4_pf_p=$?; tail -1 gpurun_out/b33_n4_pf_p.log | python -c "$J"
timeout 900 $TR --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --steps 3 --warmup 3 --prefill --persist --pd 1:3 --no-cpu-baseline > gpurun_out/b33_n4_pf_p_1p3d.log 2>&1; echo n4_pf_p_1p3d=$?; tail -1 gpurun_out/b33_n4_pf_p_1p3d.log | python -c "$J"
