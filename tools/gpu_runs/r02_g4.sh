# r02 call 4: full GPU suite x2 (flakiness), smoke, then the new N=1 bench (config 1, 64 sessions)
for i in 1 2; do
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g4_pytest_$i.log 2>&1; echo pytest$i=$?; tail -2 gpurun_out/g4_pytest_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g4_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/g4_smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/g4_bench_n1.log 2>&1; echo bench=$?; tail -1 gpurun_out/g4_bench_n1.log
