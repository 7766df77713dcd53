for c in 148 144 128 74; do
  FB_REFRESH_CTAS=$c timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:refresh_kernel -s 3 -c 3 --csv python scripts/profile_k1.py --batch 8 --layers 3 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' -v c=$c '{print c, $(NF-2), $NF}'
done
for b in 1 4 16; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:refresh_kernel -s 3 -c 2 --csv python scripts/profile_k1.py --batch $b --layers 3 2>/dev/null | grep -E "gpu__time" | awk -F'","' -v b=$b '{print "batch", b, $(NF-2), $NF}'
done
