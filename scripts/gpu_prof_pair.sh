mkdir -p gpurun_out
for v in pair single; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"pair_kernel|refresh_kernel" -s 1 -c 1 -o gpurun_out/c5_$v -f python scripts/prof_pair.py $v c5 > gpurun_out/ncu_c5_$v.log 2>&1; echo "ncu $v rc=$?"; tail -2 gpurun_out/ncu_c5_$v.log
done
