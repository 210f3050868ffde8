# r02 call 33 (2 GPUs): copy-engine job releases as one batched stream memory operation -- the copy-mode
# tests, and the block-major copy-engine lines again
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "copy or block_major or staged or ce" > gpurun_out/g33_pytest.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/g33_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pool-layout block --k1 ce > gpurun_out/g33_n1_block_ce.log 2>&1; echo n1=$?; tail -n 1 gpurun_out/g33_n1_block_ce.log | cut -c1-160
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-capped --no-cpu-baseline --pool-layout block --k1 ce --k2 ce > gpurun_out/g33_n2_block_ce.log 2>&1; echo n2=$?; tail -n 1 gpurun_out/g33_n2_block_ce.log | cut -c1-160
