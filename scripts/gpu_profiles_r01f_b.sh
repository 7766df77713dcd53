mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/k8_launches_r01f.csv python scripts/prof_k8.py > /dev/null 2>&1; echo "k8 launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 3 -c 1 -o gpurun_out/k8_gather10_vprod -f python scripts/prof_k8.py > /dev/null 2>&1; echo "k8 full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 1 -c 1 -o gpurun_out/paged_k1_b16 -f python scripts/prof_paged.py > /dev/null 2>&1; echo "paged rc=$?"
