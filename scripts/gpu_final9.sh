# r02zg: C5 launch list of the final code (K2 in row chunks) and the DRAM bytes of one whole K2 call
O=gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:skp:: -c 800 --csv --log-file $O/r02zg_c5_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo ncu rc=$?
python scripts/summarize_ncu.py launches $O/r02zg_c5_launches.csv $O/r02zg_launches_c5.txt; head -12 $O/r02zg_launches_c5.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pair -s 284 -c 142 --csv --log-file $O/r02zg_c5_k2_dram.csv python scripts/sketch_time.py 1048576 32768 8000 > /dev/null 2>&1; echo ncu2 rc=$?
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02zg_c5_k2_dram.csv')) if len(r)>5]
tot={}
n=0
for r in rows:
    name,unit,val=r[-3],r[-2],r[-1]
    try: v=float(val.replace(',',''))
    except: continue
    tot[name]=tot.get(name,0)+v; n+=1
print(n, tot)
P
