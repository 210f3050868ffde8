# r02 call 7 (2 GPUs): cross-GPU DE path tests, N=2 bench via plain `python bench.py --gpus 2`
# (self-relaunch, dual vs 1-path + storage-capped config 2), layerwise handoff TTFT,
# config-4 interference with the staged loaders, K3 NVLink counters
nvidia-smi topo -m > gpurun_out/g7_topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "peer_gpu or staged or four_gpus" > gpurun_out/g7_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g7_pytest.log
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/g7_bench_n2.log 2>&1; echo bench2=$?; tail -1 gpurun_out/g7_bench_n2.log | cut -c1-300
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g7_bench_n2_pf_lw.log 2>&1; echo pflw=$?
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline --no-layerwise > gpurun_out/g7_bench_n2_pf_nolw.log 2>&1; echo pfnolw=$?
timeout 900 python tools/interference.py --only-staged --skip-layerwise --gemms 2000 > gpurun_out/g7_interference.json 2> gpurun_out/g7_interference.err; echo interf=$?
timeout 600 python tools/prof_kernels.py --k3 --k3-tma both --k3-ctas 0,148,592 --peer --reps 3 > gpurun_out/g7_k3.json 2>&1; echo k3=$?; cat gpurun_out/g7_k3.json | cut -c1-600
timeout 900 ncu --devices 0 --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:kv_prefill_handoff -c 4 --csv --log-file gpurun_out/g7_k3_nvl.csv python tools/prof_kernels.py --k3 --k3-tma both --reps 1 > gpurun_out/g7_k3_ncu.log 2>&1; echo k3ncu=$?
