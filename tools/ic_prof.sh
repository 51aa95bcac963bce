# Per-kernel ncu durations of one bench layer in the unprotected (0), FIC (2) and IC (4) plans
for L in 0 4 8 13; do for C in 0 2 4; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python tools/variant_profile.py --layer $L --checks $C --iters 10 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki][:60]].append(float(r[vi]))
print('L$L C$C', {k:(len(v), round(sorted(v)[len(v)//2]/1000,2)) for k,v in d.items()})
"
done; done
