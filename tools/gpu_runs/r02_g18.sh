# r02 call 18 (4 GPUs): the N=4 lines on the final code -- 2P2D default line (+ 1-path, + config 2 capped),
# 1P3D, config 3 (Qwen2.5-32B KV), the full pipeline in the storage-bound regime; the 4-GPU tests
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/g18_topo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "four_gpus or 2p2d or one_queue" > gpurun_out/g18_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g18_pytest.log
timeout 1800 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g18_bench_n4.log 2>&1; echo n4=$?; tail -n 1 gpurun_out/g18_bench_n4.log | cut -c1-200
timeout 1200 python bench.py --gpus 4 --pd 1:3 --steps 3 --warmup 3 --no-capped --no-cpu-baseline > gpurun_out/g18_bench_n4_1p3d.log 2>&1; echo n4_1p3d=$?; tail -n 1 gpurun_out/g18_bench_n4_1p3d.log | cut -c1-200
timeout 1500 python bench.py --gpus 4 --workload c3 --steps 3 --warmup 3 --no-capped --no-cpu-baseline > gpurun_out/g18_bench_n4_c3.log 2>&1; echo n4c3=$?; tail -n 1 gpurun_out/g18_bench_n4_c3.log | cut -c1-200
timeout 1800 python bench.py --gpus 4 --cap-gbps 6.25 --handoff --prefill --persist --persist-mode staged --steps 3 --warmup 3 --no-capped --no-cpu-baseline > gpurun_out/g18_bench_n4_pipeline_capped.log 2>&1; echo pipe=$?; tail -n 1 gpurun_out/g18_bench_n4_pipeline_capped.log | cut -c1-200
timeout 900 python bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/g18_ref_n4.log 2>&1; echo ref4=$?; tail -n 1 gpurun_out/g18_ref_n4.log | cut -c1-200
