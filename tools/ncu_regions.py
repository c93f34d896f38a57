"""Group an ncu --set full capture's SASS into execution-count regions and
report instruction share, sampled stall share and the top stall reasons per
region (the source page must have been captured with --import-source on).

    python tools/ncu_regions.py capture.ncu-rep [> summary.txt]
"""
import csv, sys, subprocess
rep=sys.argv[1]
subprocess.run(f"ncu -i {rep} --page source --csv --print-source sass > /tmp/_ncu_src.csv 2>/dev/null", shell=True)
subprocess.run(f"ncu -i {rep} --page raw --csv > /tmp/_ncu_raw.csv 2>/dev/null", shell=True)
rows=list(csv.reader(open('/tmp/_ncu_raw.csv'))); d=dict(zip(rows[0],rows[2]))
for k in ['gpu__time_duration.sum','smsp__inst_executed.sum','sm__issue_active.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed']:
    print(k, d.get(k))
rows=list(csv.reader(open('/tmp/_ncu_src.csv')))
h=rows[1]; data=rows[2:]
iS=h.index('Warp Stall Sampling (All Samples)'); iE=h.index('Instructions Executed'); iSrc=h.index('Source')
cols=[c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot_s=sum(int(r[iS] or 0) for r in data); tot_e=sum(int(r[iE] or 0) for r in data)
print('samples',tot_s,'inst',tot_e)
# regions: split by execution count changes
reg=[]; cur=None
for i,r in enumerate(data):
    e=int(r[iE] or 0)
    if cur is None or abs(e-cur[2])>0.05*max(e,cur[2],1):
        cur=[i,i,e]; reg.append(cur)
    else: cur[1]=i
for a,b,e in reg:
    s=sum(int(data[i][iS] or 0) for i in range(a,b+1))
    if s<0.01*tot_s and e*(b-a+1)<0.01*tot_e: continue
    st={c.replace('stall_',''):sum(int(data[i][h.index(c)] or 0) for i in range(a,b+1)) for c in cols}
    st={k:v for k,v in sorted(st.items(), key=lambda x:-x[1])[:5] if v>0}
    print(f"[{a:5d}-{b:5d}] n={b-a+1:4d} exec/inst={e:8d} inst%={100*e*(b-a+1)/tot_e:5.1f} samp%={100*s/tot_s:5.1f} {st}  first: {data[a][iSrc].strip()[:50]}")
