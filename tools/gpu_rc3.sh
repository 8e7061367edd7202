mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"redchain|red_|ew_vec" --csv --log-file gpurun_out/rc_launch.csv python tools/redchain_bench.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/rc_launch.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki][:40]), {})[r[mi]]=float(r[vi].replace(',',''))
for (i,k),m in sorted(d.items())[:400:4]:
    t=m.get('gpu__time_duration.sum',0); b=m.get('dram__bytes_read.sum',0)
    print(f"{i:5d} {k:40s} {t/1e3:8.1f} us {b/1e6:8.1f} MB {b/t if t else 0:7.0f} GB/s")
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:redchain_cols -s 6 -c 1 -o gpurun_out/rc_cols -f python tools/redchain_bench.py > /dev/null 2>&1
ncu -i gpurun_out/rc_cols.ncu-rep --page details --csv > gpurun_out/rc_cols_details.csv 2>&1
grep -i "stall\|Warp Cycles\|Occupancy\|Throughput\|Eligible\|Issued" gpurun_out/rc_cols_details.csv | head -40
rm -f gpurun_out/rc_launch.csv
