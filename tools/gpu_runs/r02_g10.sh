# r02 call 10 (2 GPUs): full suite, kernel smoke of every kernel, K3 rate, interference, N=2 line,
# layerwise handoff (batched per forward) vs after-forward, online APS capacity (live mode)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g10_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g10_pytest.log
timeout 300 python tools/sanitize/kernels_small.py > gpurun_out/g10_kernels_small.log 2>&1; echo small=$?; tail -1 gpurun_out/g10_kernels_small.log
timeout 600 python tools/prof_kernels.py --k3 --k3-tma both --peer --reps 3 > gpurun_out/g10_k3.json 2>&1; echo k3=$?; cut -c1-400 gpurun_out/g10_k3.json
timeout 900 python tools/interference.py --only-staged --skip-layerwise --gemms 2000 > gpurun_out/g10_interference.json 2> gpurun_out/g10_interference.err; echo interf=$?
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/g10_bench_n2.log 2>&1; echo bench2=$?; tail -1 gpurun_out/g10_bench_n2.log | cut -c1-200
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g10_pf_lw.log 2>&1; echo pflw=$?
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline --no-layerwise > gpurun_out/g10_pf_nolw.log 2>&1; echo pfnolw=$?
timeout 1500 python tools/online_capacity.py --pd 1:1 --sessions 48 --turns 8 --cap-gbps 6.25 --slo 2.0 --bisect 2 > gpurun_out/g10_online.json 2> gpurun_out/g10_online.err; echo online=$?; tail -2 gpurun_out/g10_online.err
