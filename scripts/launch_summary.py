import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0,0.0])
for r in rows[hdr_i+1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('ttg::<unnamed>::','').replace('void ','')
    v = float(r[vi].replace(',',''))
    unit = r[ui]
    v *= {'nsecond':1,'usecond':1e3,'msecond':1e6,'second':1e9}.get(unit,1)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{k[:50]:50s} n={v[0]:5d} total={v[1]/1e6:9.3f} ms  share={v[1]/tot:.3f}")
print("total kernel ms", round(tot/1e6,3), "launches", sum(v[0] for v in agg.values()))
