# r02 call 16 (2 GPUs): copy-engine K3 + after-forward handoff as defaults, staged K4 executor cases,
# live prefill + handoff, K4 ceiling into the store's own pages, online capacity with first-token TTFT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g16_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g16_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g16_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g16_smoke.log
timeout 400 python tools/prof_kernels.py --k4 > gpurun_out/g16_k4.json 2> gpurun_out/g16_k4.err; echo prof=$?; cat gpurun_out/g16_k4.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g16_pf.log 2>&1; echo pf=$?; tail -n 1 gpurun_out/g16_pf.log | cut -c1-200
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --persist --persist-mode staged --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g16_pf_persist.log 2>&1; echo pfp=$?; tail -n 1 gpurun_out/g16_pf_persist.log | cut -c1-200
timeout 1500 python tools/online_capacity.py --pd 1:1 --prefill --handoff --bisect 2 > gpurun_out/g16_online_handoff.json 2> gpurun_out/g16_online_handoff.err; echo onlineh=$?; tail -n 2 gpurun_out/g16_online_handoff.err
