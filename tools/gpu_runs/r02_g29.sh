# r02 call 29 (2 GPUs): online APS capacity with the reference's first-token TTFT on 256 sessions, so the
# dual path's capacity is reached inside the search (96 sessions never violated up to 256 sessions/s)
mkdir -p gpurun_out
timeout 2700 python tools/online_capacity.py --pd 1:1 --prefill --handoff --slo 1.0 --sessions 256 --aps-max 1024 --bisect 2 > gpurun_out/g29_online_256.json 2> gpurun_out/g29_online_256.err; echo online=$?; tail -n 3 gpurun_out/g29_online_256.err
