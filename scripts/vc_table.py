"""Dev tool: per-kernel table of the last V-cycle in an ncu launch CSV (see vcycle_profile.py)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hdr_i]; ix = {h: i for i, h in enumerate(hdr)}
recs = {}
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr): continue
    d = recs.setdefault(r[ix['ID']], {'name': r[ix['Kernel Name']][:46]})
    d[r[ix['Metric Name']]] = (r[ix['Metric Value']], r[ix['Metric Unit']])
ids = sorted(recs, key=int)
last = [i for i in ids if 'project_kernel' in recs[i]['name']][-1]
tot = 0.0
for i in ids[ids.index(last):]:
    v, u = recs[i]['gpu__time_duration.sum']
    t = float(v.replace(',', '')) / (1000.0 if u == 'ns' else 1.0)
    tot += t
    print(f"{recs[i]['name']:48s} grid {recs[i].get('launch__grid_size', ('?',))[0]:>6s} {t:8.1f} us")
print(f"total {tot:.1f} us")
