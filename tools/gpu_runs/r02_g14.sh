# r02 call 14 (2 GPUs): redo call 12's lost evidence on HEAD (full 2-GPU suite, interference A/B/A,
# layerwise vs after-forward handoff, online APS capacity) + NVLink copy-engine probe + K3 alone
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/g14_topo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g14_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g14_pytest.log
timeout 300 python tools/probe_nvlink.py > gpurun_out/g14_probe_nvlink.json 2> gpurun_out/g14_probe_nvlink.err; echo probe=$?; cat gpurun_out/g14_probe_nvlink.json | cut -c1-600
timeout 300 python tools/prof_kernels.py --k3 --peer > gpurun_out/g14_k3.json 2> gpurun_out/g14_k3.err; echo k3=$?; cat gpurun_out/g14_k3.json
timeout 1200 python tools/interference.py --only-staged --skip-layerwise --gemms 3000 > gpurun_out/g14_interference.json 2> gpurun_out/g14_interference.err; echo interf=$?
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g14_pf_lw.log 2>&1; echo pflw=$?; tail -n 1 gpurun_out/g14_pf_lw.log | cut -c1-300
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline --no-layerwise > gpurun_out/g14_pf_nolw.log 2>&1; echo pfnolw=$?; tail -n 1 gpurun_out/g14_pf_nolw.log | cut -c1-300
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --k3 ce --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g14_pf_lw_k3ce.log 2>&1; echo pflwce=$?; tail -n 1 gpurun_out/g14_pf_lw_k3ce.log | cut -c1-300
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g14_ho.log 2>&1; echo ho=$?; tail -n 1 gpurun_out/g14_ho.log | cut -c1-300
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --k3 ce --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g14_ho_k3ce.log 2>&1; echo hoce=$?; tail -n 1 gpurun_out/g14_ho_k3ce.log | cut -c1-300
timeout 2000 python tools/online_capacity.py --pd 1:1 --bisect 2 > gpurun_out/g14_online.json 2> gpurun_out/g14_online.err; echo online=$?; tail -n 2 gpurun_out/g14_online.err
