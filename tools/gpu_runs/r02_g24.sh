# r02 call 24 (4 GPUs): config 5 on the final code -- online (Poisson) arrivals in plan mode, asymmetric
# per-engine storage caps, the scheduler's load balance (load_balance_ratio), at 2 and 4 GPUs
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --online 2 --caps 6.25,3.125 --sessions-per-gpu 4 --no-cpu-baseline > gpurun_out/g24_n2_c5.log 2>&1; echo n2c5=$?; tail -n 1 gpurun_out/g24_n2_c5.log | cut -c1-200
timeout 1200 python bench.py --gpus 4 --steps 3 --warmup 3 --online 4 --caps 6.25,3.125,6.25,3.125 --sessions-per-gpu 4 --no-cpu-baseline > gpurun_out/g24_n4_c5.log 2>&1; echo n4c5=$?; tail -n 1 gpurun_out/g24_n4_c5.log | cut -c1-200
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "four_gpus" > gpurun_out/g24_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g24_pytest.log
