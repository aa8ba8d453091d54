import csv, json, sys, glob
for f in sys.argv[1:]:
    if f.endswith('.log'):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(f, round(d['value']/1e9, 3), 'G/s', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['frac'], 3), d['clocks'])
        except Exception as e:
            print(f, 'ERR', open(f).read()[-500:])
    else:
        rows = list(csv.reader(open(f)))
        hdr = None; data = {}
        for r in rows:
            if r and r[0] == 'ID': hdr = r; continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                data.setdefault((int(d['ID']), d['Kernel Name'][:46]), {})[d['Metric Name']] = d['Metric Value']
        for k, v in sorted(data.items()):
            t = float(v.get('gpu__time_duration.sum', 0)) / 1e3
            rd = float(v.get('dram__bytes_read.sum', 0)) / 1e9
            wr = float(v.get('dram__bytes_write.sum', 0)) / 1e9
            print(k[0], k[1], f"{t:8.1f} us  R {rd:6.2f} GB W {wr:6.2f} GB  {((rd+wr)/(t*1e-6)/1e3) if t else 0:6.0f} GB/s",
                  {kk: vv for kk, vv in v.items() if kk.startswith(('launch', 'sm__'))})
