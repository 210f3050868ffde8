# r02 call 22 (2 GPUs): final full 2-GPU suite, the default N=2 line, layerwise handoff with the
# copy-engine K3 gated by stream waits vs after the forward
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g22_pytest.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/g22_pytest.log
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g22_bench_n2.log 2>&1; echo n2=$?; tail -n 1 gpurun_out/g22_bench_n2.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --layerwise --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g22_pf_lw_memop.log 2>&1; echo pflw=$?; tail -n 1 gpurun_out/g22_pf_lw_memop.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g22_pf.log 2>&1; echo pf=$?; tail -n 1 gpurun_out/g22_pf.log | cut -c1-200
