# r02 call 38 (4 GPUs): link peaks of every GPU -- H2D alone / concurrent, the NVLink copy-engine matrix
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/g38_topo.txt 2>&1
timeout 600 python tools/probe_links_all.py > gpurun_out/g38_links.json 2> gpurun_out/g38_links.err; echo links=$?; cat gpurun_out/g38_links.json
