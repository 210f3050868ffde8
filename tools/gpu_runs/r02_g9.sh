# r02 call 9 (2 GPUs): copy-engine scatter, buffer bound, live mode; interference; N=2 / N=1 benches; sanitizers
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "staged or buffer or live or handoff or tma" > gpurun_out/g9_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/g9_pytest.log
timeout 900 python tools/interference.py --only-staged --skip-layerwise --gemms 2000 > gpurun_out/g9_interference.json 2> gpurun_out/g9_interference.err; echo interf=$?; tail -2 gpurun_out/g9_interference.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 3 --warmup 2 --stage-scatter ce --no-cpu-baseline > gpurun_out/g9_bench_n1_ce.log 2>&1; echo n1ce=$?; tail -1 gpurun_out/g9_bench_n1_ce.log | cut -c1-200
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 2 --stage-scatter ce --no-cpu-baseline > gpurun_out/g9_bench_n2_ce.log 2>&1; echo n2ce=$?; tail -1 gpurun_out/g9_bench_n2_ce.log | cut -c1-200
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 2 --stage-ctas 148 --no-capped --no-cpu-baseline > gpurun_out/g9_bench_n2_k148.log 2>&1; echo n2k148=$?; tail -1 gpurun_out/g9_bench_n2_k148.log | cut -c1-200
bash tools/gpu_runs/r02_g8.sh
