# r02 call 31 (2 GPUs): block-major PE pools -- kernel / copy-engine parity, the executor, then the
# loaders straight into them by the copy engines: N=1 and N=2 lines, and their interference
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "block_major" > gpurun_out/g31_pytest.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/g31_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool-layout block --k1 ce > gpurun_out/g31_n1_block_ce.log 2>&1; echo n1=$?; tail -n 1 gpurun_out/g31_n1_block_ce.log | cut -c1-200
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-capped --no-cpu-baseline --pool-layout block --k1 ce --k2 ce > gpurun_out/g31_n2_block_ce.log 2>&1; echo n2=$?; tail -n 1 gpurun_out/g31_n2_block_ce.log | cut -c1-200
timeout 1200 python tools/interference.py --skip-layerwise --gemms 3000 --block-major > gpurun_out/g31_interference_block.json 2> gpurun_out/g31_interference_block.err; echo interf=$?; tail -n 2 gpurun_out/g31_interference_block.err
