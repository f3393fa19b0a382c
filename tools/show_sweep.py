import csv, collections, sys
rows = list(csv.DictReader(open(sys.argv[1])))
t = collections.defaultdict(dict)
for r in rows:
    t[(r['op'], int(r['bytes']))][r['algorithm']] = (float(r['median_us']), float(r['busbw_gbs']))
for (op, b), d in sorted(t.items()):
    print(f"{op:12s} {b:>11d} " + "  ".join(f"{a}:{v[0]:8.1f}us {v[1]:6.1f}" for a, v in sorted(d.items())))
