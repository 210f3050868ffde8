# r02 call 39 (2 GPUs): config 5 in live mode -- asymmetric storage caps (6.25 / 3.125 GB/s), Poisson
# arrivals, the reference's first-token TTFT (SLO 1 s), 128 sessions
mkdir -p gpurun_out
timeout 660 python tools/online_capacity.py --pd 1:1 --caps 6.25,3.125 --prefill --handoff --slo 1.0 --sessions 128 --aps-start 4 --aps-max 256 --bisect 1 > gpurun_out/g39_online_c5.json 2> gpurun_out/g39_online_c5.err; echo online=$?; tail -n 2 gpurun_out/g39_online_c5.err
