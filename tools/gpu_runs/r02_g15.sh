# r02 call 15 (2 GPUs): K3 on the copy engines with the miss KV overlapped, staged K4, live prefill;
# the layerwise-handoff hang of g14 (rank 1 watchdog) bisected: 64 vs 148 K3 CTAs, longer watchdog
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g15_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g15_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g15_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g15_smoke.log
timeout 400 python tools/prof_kernels.py --k3 --k4 --peer > gpurun_out/g15_k3k4.json 2> gpurun_out/g15_k3k4.err; echo prof=$?; cat gpurun_out/g15_k3k4.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --handoff-ctas 64 --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g15_pf_lw64.log 2>&1; echo pflw64=$?; tail -n 1 gpurun_out/g15_pf_lw64.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --wait-timeout-ms 90000 --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g15_pf_lw148.log 2>&1; echo pflw148=$?; tail -n 1 gpurun_out/g15_pf_lw148.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --persist --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g15_persist_k4.log 2>&1; echo pk4=$?; tail -n 1 gpurun_out/g15_persist_k4.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --persist --persist-mode staged --k3 ce --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g15_persist_staged.log 2>&1; echo pst=$?; tail -n 1 gpurun_out/g15_persist_staged.log | cut -c1-200
timeout 1500 python tools/online_capacity.py --pd 1:1 --prefill --bisect 2 > gpurun_out/g15_online_prefill.json 2> gpurun_out/g15_online_prefill.err; echo onlinep=$?; tail -n 2 gpurun_out/g15_online_prefill.err
