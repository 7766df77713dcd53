mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/k8_launches.csv python scripts/prof_k8.py > gpurun_out/k8.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows=list(csv.DictReader(open('gpurun_out/k8_launches.csv')))
for r in rows:
    if r.get('Metric Name') in ('gpu__time_duration.sum','dram__bytes_read.sum'):
        print(r['Kernel Name'][:60], r['Metric Name'], r['Metric Value'], r['Metric Unit'])
PY
