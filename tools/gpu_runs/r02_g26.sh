# r02 call 26 (2 GPUs): the copy-engine K3 pushing the whole prompt from the PE pool (the side kernel
# now writes the miss KV locally) -- its tests, K3 alone, the handoff pipeline, the one-queue runs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "handoff or copy_engine or live or one_queue or prefill" > gpurun_out/g26_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g26_pytest.log
timeout 400 python tools/prof_kernels.py --k3 --peer > gpurun_out/g26_k3.json 2> gpurun_out/g26_k3.err; echo k3=$?; cat gpurun_out/g26_k3.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --handoff --prefill --persist --no-capped --no-one-path --no-cpu-baseline > gpurun_out/g26_pf_persist.log 2>&1; echo pfp=$?; tail -n 1 gpurun_out/g26_pf_persist.log | cut -c1-200
