import csv, collections, re, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[hi]
k=h.index('Kernel Name'); v=h.index('Metric Value')
tot=collections.Counter(); cnt=collections.Counter()
for r in rows[hi+1:]:
    if len(r)>v:
        nm=r[k].replace('(anonymous namespace)','anon')
        m=re.search(r'([A-Za-z_][A-Za-z0-9_]*)\s*(<[^()]*>)?\s*\(', nm)
        name=m.group(1) if m else nm[:30]
        tot[name]+=float(r[v].replace(',','')); cnt[name]+=1
for n,t in tot.most_common(6): print(f"{n:24s} {cnt[n]:5d} {t/1e3:10.1f} us")
