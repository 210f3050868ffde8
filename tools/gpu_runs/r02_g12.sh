# r02 call 12 (2 GPUs): new tests (dual staged, PersistWrite, attend signal, copy-engine per job),
# interference incl. per-job copy-engine loaders, layerwise handoff v3 vs after-forward, online APS capacity
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g12_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g12_pytest.log
timeout 900 python tools/interference.py --only-staged --skip-layerwise --gemms 2000 > gpurun_out/g12_interference.json 2> gpurun_out/g12_interference.err; echo interf=$?
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g12_pf_lw.log 2>&1; echo pflw=$?
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline --no-layerwise > gpurun_out/g12_pf_nolw.log 2>&1; echo pfnolw=$?
timeout 1200 python bench.py --gpus 2 --steps 2 --warmup 1 --k1 ce --k2 ce --no-capped --no-cpu-baseline > gpurun_out/g12_bench_n2_ce_job.log 2>&1; echo n2ce=$?
timeout 2400 python tools/online_capacity.py --pd 1:1 --bisect 3 > gpurun_out/g12_online.json 2> gpurun_out/g12_online.err; echo online=$?; tail -2 gpurun_out/g12_online.err
