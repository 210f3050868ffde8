# r02 call 37 (2 GPUs): one ncu --set full capture each of the copy-engine K3's side kernel and of the staged
# K4's gather (kv_persist_d2h into the HBM ring)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kv_handoff_side" -c 1 -o gpurun_out/g37_side python tools/prof_kernels.py --k3 --reps 1 > gpurun_out/g37_side.log 2>&1; echo side=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kv_persist_d2h" -c 1 -o gpurun_out/g37_persist python tools/prof_kernels.py --k4 --reps 1 --jobs 8 > gpurun_out/g37_persist.log 2>&1; echo persist=$?
ls -la gpurun_out/g37_*
