timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest16.log 2>&1; echo pytest=$?; tail -25 gpurun_out/pytest16.log
