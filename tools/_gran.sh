mkdir -p gpurun_out
./tools/gran_probe 0 | head -3
for L in 32 64; do
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv ./tools/gran_probe $L > gpurun_out/gran3_$L.csv 2>&1; echo ncu=$?
grep "limit\|set Max" gpurun_out/gran3_$L.csv
python3 - $L <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f"gpurun_out/gran3_{sys.argv[1]}.csv")) if len(r)>12 and "probe" in r[4]]
d={}
for r in rows: d.setdefault(r[4].split("(")[0],{})[r[12]]=r[14]
for k,v in d.items(): print(k, v)
PY
done
