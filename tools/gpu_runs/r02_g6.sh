# r02 call 6: full 1-GPU suite + smoke + default N=1 bench (staged K1) + ncu launch list + scatter capture
nvidia-smi topo -m > gpurun_out/g6_topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g6_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g6_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g6_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/g6_smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/g6_bench_n1.log 2>&1; echo bench=$?; tail -1 gpurun_out/g6_bench_n1.log | cut -c1-400
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g6_ref_n1.log 2>&1; echo ref=$?; tail -1 gpurun_out/g6_ref_n1.log | cut -c1-300
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g6_launches_n1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g6_ncu_list.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather --launch-skip 200 -c 1 -o gpurun_out/g6_scatter_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/g6_ncu_full.log 2>&1; echo ncu_full=$?
