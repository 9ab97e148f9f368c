import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','details','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
hdr=r[0]
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); ui=hdr.index('Metric Unit'); vi=hdr.index('Metric Value')
want=['Duration','DRAM Throughput','L1/TEX Hit Rate','L2 Hit Rate','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','Executed Ipc Active','Issue Slots Busy','Warp Cycles Per Issued Instruction','Executed Instructions','Memory Throughput','Max Bandwidth','L1/TEX Cache Throughput','L2 Cache Throughput','Mem Pipes Busy']
for row in r[1:]:
  if row[mi] in want: print(row[ki][:26], '|', row[mi], '=', row[vi], row[ui])
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines()))
hdr=r[0]
for row in r[2:]:
  d=dict(zip(hdr,row))
  for k in ['dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','l1tex__t_bytes.sum','gpu__time_duration.sum']:
    print(k, d.get(k), r[1][hdr.index(k)] if k in hdr else '')
  st=[(h,v) for h,v in d.items() if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
  def f(v):
    try: return float(v.replace(',',''))
    except: return 0
  print(sorted([(f(v),h.replace('smsp__pcsamp_warps_issue_stalled_','')) for h,v in st],reverse=True)[:8])
