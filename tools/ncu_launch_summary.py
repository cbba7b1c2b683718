import csv,sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=defaultdict(dict)
for r in rows[hdr+1:]:
    d[int(r[ii])][r[mi]]=float(r[vi].replace(',',''))
    d[int(r[ii])]['name']=r[ki].split('(')[0].replace('void ','').replace('unnamed>::','')
agg=defaultdict(list)
for i,v in sorted(d.items()):
    agg[v['name']].append((v['gpu__time_duration.sum'],v['dram__bytes_read.sum']+v['dram__bytes_write.sum']))
for n,l in agg.items():
    import statistics
    t=statistics.median(x[0] for x in l); b=statistics.median(x[1] for x in l)
    print(f"{n:45s} launches={len(l):3d} median_ns={t:9.0f} dram_bytes={b:12.0f} GB/s={b/t:7.1f}")
