timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest35.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest35.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 120 python tools/prof_k5.py > gpurun_out/k5b.txt 2>&1 && cat gpurun_out/k5b.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_prefill_attend -s 3 -c 1 -o gpurun_out/r01_k5b_full -f python tools/prof_k5.py > gpurun_out/k5b_ncu.log 2>&1; echo ncu=$?
