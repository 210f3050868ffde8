# r02 call 19 (2 GPUs): staged K4 as the default (persistence tests), online capacity with the
# first-token TTFT and 100 GB pools (g17's outliers were decode-pool admission stalls at 4x the largest prompt)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "persist or live or one_queue" > gpurun_out/g19_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g19_pytest.log
timeout 2000 python tools/online_capacity.py --pd 1:1 --prefill --handoff --slo 1.0 --bisect 2 > gpurun_out/g19_online_handoff.json 2> gpurun_out/g19_online_handoff.err; echo onlineh=$?; tail -n 2 gpurun_out/g19_online_handoff.err
