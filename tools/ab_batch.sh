for v in old b12 b16; do
  AMGR_LIB=abtest/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/ab_$v.csv python tools/region_driver.py 256 vcycle > /dev/null 2>&1
  python - <<PY
import csv
rows = list(csv.reader(open('gpurun_out/ab_$v.csv')))
h = [i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[h]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
ks = [(r[ki], float(r[vi].replace(',',''))) for r in rows[h+1:] if len(r) > vi]
half = ks[len(ks)//2:]
rp = [round(v/1e3,1) for k,v in half if 'k_rowpass<' in k]
print('$v vcycle', round(sum(v for _,v in half)/1e3,1), rp[:5], rp[-5:])
PY
done
