# r02 call 36 (4 GPUs): online APS capacity at 2P2D (live mode: the global scheduler balancing 2 PEs and 2 DEs),
# the reference's first-token TTFT, 6.25 GB/s caps, 256 sessions
mkdir -p gpurun_out
timeout 2400 python tools/online_capacity.py --pd 2:2 --prefill --handoff --slo 1.0 --sessions 256 --aps-start 8 --aps-max 1024 --bisect 1 > gpurun_out/g36_online_2p2d.json 2> gpurun_out/g36_online_2p2d.err; echo online=$?; tail -n 3 gpurun_out/g36_online_2p2d.err
