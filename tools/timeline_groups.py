import csv, sys
R=list(csv.DictReader(open(sys.argv[1])))
for r in R: r['t0']=float(r['t0']); r['t1']=float(r['t1']); r['stream']=int(r['stream'])
wall=max(r['t1'] for r in R)
for g in range(4):
    rs=[r for r in R if r['stream'] in (2*g, 2*g+1)]
    if not rs: continue
    big=[r for r in rs if r['cls']=='zgemm' and float(r['flops'])>2e9]
    lastbig=max(r['t1'] for r in big) if big else 0
    print(f"group {g}: first {min(r['t0'] for r in rs):.3f} last big GEMM end {lastbig:.3f} last launch end {max(r['t1'] for r in rs):.3f}")
print("wall", wall)
