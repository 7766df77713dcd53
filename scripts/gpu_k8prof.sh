mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"refresh_kernel" -s 3 -c 1 -o gpurun_out/k8_gather10 -f python scripts/prof_k8.py > gpurun_out/k8prof.log 2>&1; echo "rc=$?"
