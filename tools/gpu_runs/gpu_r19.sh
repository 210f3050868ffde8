timeout 300 ./tools/probe_ce > gpurun_out/probe_ce2.txt 2>&1; echo probe=$?
timeout 600 python bench.py --steps 5 --warmup 3 --k1 ce --no-cpu-baseline > gpurun_out/b19_ce.log 2>&1; echo ce=$?; tail -1 gpurun_out/b19_ce.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b19_sm.log 2>&1; echo sm=$?; tail -1 gpurun_out/b19_sm.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest19.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest19.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
