import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == 'ID':
        hdr = r; start = i; break
idx = {h: i for i, h in enumerate(hdr)}
agg = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr): continue
    agg.setdefault((int(r[idx['ID']]), r[idx['Kernel Name']][:48]), {})[r[idx['Metric Name']]] = float(r[idx['Metric Value']].replace(',', ''))
for (i, n), m in sorted(agg.items()):
    t = m.get('gpu__time_duration.sum', 0); rb = m.get('dram__bytes_read.sum', 0); wb = m.get('dram__bytes_write.sum', 0)
    print(i, n, f"{t/1000:.1f}us rd={rb/1e6:.1f}MB wr={wb/1e6:.1f}MB {((rb+wb)/t):.0f}GB/s" if t else "")
