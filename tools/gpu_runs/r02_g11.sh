# r02 call 11 (4 GPUs): N=4 lines (2P2D + config 2 capped; 1P3D; Qwen config 3), the full pipeline in the
# storage-bound regime, the 4-GPU tests
nvidia-smi topo -m > gpurun_out/g11_topo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "four_gpus or 2p2d" > gpurun_out/g11_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/g11_pytest.log
timeout 1800 python bench.py --gpus 4 --steps 3 --warmup 2 > gpurun_out/g11_bench_n4.log 2>&1; echo n4=$?; tail -1 gpurun_out/g11_bench_n4.log | cut -c1-160
timeout 1200 python bench.py --gpus 4 --pd 1:3 --steps 2 --warmup 1 --no-capped --no-cpu-baseline > gpurun_out/g11_bench_n4_1p3d.log 2>&1; echo n4_1p3d=$?
timeout 1500 python bench.py --gpus 4 --workload c3 --steps 2 --warmup 1 --no-capped --no-cpu-baseline > gpurun_out/g11_bench_n4_c3.log 2>&1; echo n4c3=$?
timeout 1800 python bench.py --gpus 4 --cap-gbps 6.25 --handoff --prefill --persist --steps 2 --warmup 1 --no-capped --no-cpu-baseline > gpurun_out/g11_bench_n4_pipeline_capped.log 2>&1; echo pipe=$?
