timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest47.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest47.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/b47_n1.log 2>&1; echo n1=$?; tail -1 gpurun_out/b47_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline'], d['clocks'])"
