# r02 call 20 (1 GPU, the driver's round-end box): final code -- pytest -m gpu, smoke, bench N=1 both
# arms, the ncu launch list of the bench, one ncu --set full of the K3 side kernel / staged K4 gather
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g20_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g20_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g20_smoke.log 2>&1; echo smoke=$?; tail -n 1 gpurun_out/g20_smoke.log
timeout 900 python bench.py > gpurun_out/g20_bench_n1.log 2>&1; echo n1=$?; tail -n 1 gpurun_out/g20_bench_n1.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/g20_ref_n1.log 2>&1; echo ref=$?; tail -n 1 gpurun_out/g20_ref_n1.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g20_launches_n1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g20_ncu.log 2>&1; echo ncu=$?
