# r02 call 27 (2 GPUs): the copy-engine K3 after g26 (gated calls keep the miss KV in the side kernel):
# the handoff / copy-engine / live / one-queue / prefill tests, K3 alone, the pipeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "handoff or copy_engine or live or one_queue or prefill" > gpurun_out/g27_pytest.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/g27_pytest.log
timeout 400 python tools/prof_kernels.py --k3 --peer > gpurun_out/g27_k3.json 2> gpurun_out/g27_k3.err; echo k3=$?; cat gpurun_out/g27_k3.json
