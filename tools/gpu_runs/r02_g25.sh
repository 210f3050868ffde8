# r02 call 25 (2 GPUs): K1 staged interference vs the HBM ring size (an L2-sized ring keeps the ring
# traffic out of HBM), and the N=1 line's rate at those ring sizes
mkdir -p gpurun_out
timeout 1200 python tools/interference.py --skip-layerwise --gemms 3000 --ring-mb 1024,256,64,32 > gpurun_out/g25_ring.json 2> gpurun_out/g25_ring.err; echo ring=$?; tail -n 2 gpurun_out/g25_ring.err
for r in 64 32; do CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --stage-ring-mb $r > gpurun_out/g25_n1_ring$r.log 2>&1; echo n1_$r=$?; tail -n 1 gpurun_out/g25_n1_ring$r.log | cut -c1-160; done
