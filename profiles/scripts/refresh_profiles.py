"""Copy the final measurement pass (gpurun_out/f_*) into profiles/ and print the tables."""
import csv, io, json, os, subprocess, collections
R = '/root/repo'
G = f'{R}/gpurun_out'
P = f'{R}/profiles'

def last_json(path):
    lines = [l for l in open(path).read().strip().splitlines() if l.startswith('{')]
    return json.loads(lines[-1])

for c in ['c2', 'c3', 'c4', 'c4r64', 'c5', 'c2_one', 'c2_two']:
    f = f'{G}/f_bench_{c}.json'
    if os.path.exists(f):
        d = last_json(f)
        json.dump(d, open(f'{P}/r01_bench_{c}.json', 'w'))
d = last_json(f'{G}/f_ref_c2.json'); json.dump(d, open(f'{P}/r01_reference_c2.json', 'w'))
if os.path.exists(f'{G}/f_launches_c2.csv'):
    open(f'{P}/r01_c2_launches.csv', 'w').write(open(f'{G}/f_launches_c2.csv').read())
for src, dst in [('f_mttkrp_c2', 'r01_mttkrp_c2_ncu_raw.csv'), ('f_solve_c2', 'r01_solve_c2_ncu_raw.csv'),
                 ('f_mttkrp_c2_one', 'r01_mttkrp_c2_one_ncu_raw.csv')]:
    rep = f'{G}/{src}.ncu-rep'
    if os.path.exists(rep):
        out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
        open(f'{P}/{dst}', 'w').write(out)

traffic = {"_source": "ROOT MTTKRP DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), ncu --clock-control none: c2 from profiles/r01_mttkrp_c2_ncu_raw.csv (--set full, iteration 4 of 5, the timed gather policy), c4/c5 from `ncu --metrics ... -k regex:mttkrp_csf_kernel -c 8 python bench.py --config cX --steps 1 --warmup 0 --iters 2` (profiles/r01_traffic_cX.csv); mean over the captured launches"}
def raw_rows(path):
    rows = list(csv.reader(open(path)))
    return rows[0], rows[2:]
h, rows = raw_rows(f'{P}/r01_mttkrp_c2_ncu_raw.csv')
def num(x): return float(x.replace(',', ''))
rd = [num(r[h.index('dram__bytes_read.sum')]) for r in rows]
wr = [num(r[h.index('dram__bytes_write.sum')]) for r in rows]
hit = [num(r[h.index('lts__t_sector_hit_rate.pct')]) for r in rows]
unit = list(csv.reader(open(f'{P}/r01_mttkrp_c2_ncu_raw.csv')))[1][h.index('dram__bytes_read.sum')]
scale = {'Mbyte': 1e6, 'Gbyte': 1e9, 'Kbyte': 1e3, 'byte': 1}[unit]
b2 = json.load(open(f'{P}/r01_bench_c2.json'))
traffic['c2:G1'] = {"dram_bytes_per_launch": sum(a + b for a, b in zip(rd, wr)) / len(rd) * scale,
                    "alg_bytes_per_launch": b2['roofline']['alg_bytes_per_launch'],
                    "l2_hit_rate_pct": sum(hit) / len(hit)}
for c in ['c4', 'c5']:
    f = f'{G}/f_traffic_{c}.csv'
    if not os.path.exists(f):
        continue
    txt = open(f).read(); i = txt.index('"ID"')
    open(f'{P}/r01_traffic_{c}.csv', 'w').write(txt[i:])
    rr = list(csv.reader(io.StringIO(txt[i:]))); hh = rr[0]
    per = collections.defaultdict(dict)
    for r in rr[1:]:
        if len(r) == len(hh):
            per[r[hh.index('ID')]][r[hh.index('Metric Name')]] = (num(r[hh.index('Metric Value')]), r[hh.index('Metric Unit')])
    sc = lambda v: v[0] * {'Mbyte': 1e6, 'Gbyte': 1e9, 'Kbyte': 1e3, 'byte': 1}.get(v[1], 1)
    tot = [sc(m['dram__bytes_read.sum']) + sc(m['dram__bytes_write.sum']) for m in per.values()]
    hits = [m['lts__t_sector_hit_rate.pct'][0] for m in per.values()]
    bc = json.load(open(f'{P}/r01_bench_{c}.json'))
    traffic[f'{c}:G1'] = {"dram_bytes_per_launch": sum(tot) / len(tot),
                          "alg_bytes_per_launch": bc['roofline']['alg_bytes_per_launch'],
                          "l2_hit_rate_pct": sum(hits) / len(hits)}
json.dump(traffic, open(f'{P}/mttkrp_traffic.json', 'w'), indent=1)
print(json.dumps(traffic, indent=1)[:1500])
for c in ['c2', 'c3', 'c4', 'c4r64', 'c5', 'c2_two', 'c2_one']:
    d = json.load(open(f'{P}/r01_bench_{c}.json')); r = d['roofline']; e = (d.get('e2e') or {}).get('value')
    g = r.get('gather') or {}
    print(f"| {c} | {d['ms_per_step']:.2f} ms | {d['value']:.3g} | {d['cpals_sec_per_iter']*1e3:.2f} ms | {d['mttkrp_nnzR_per_s']:.3g} | {r['frac']:.2f} | {r.get('frac_compulsory') or 0:.3f} | {g.get('frac')} | {('%.3g' % e) if e else ''} | {d['clocks']['sm_mhz']:.0f} {','.join(d['clocks']['reasons'])} | traffic {r.get('traffic')}")
