"""Copy the round-2 final measurement pass (gpurun_out/fin_*, profiles/scripts/r02_final.sh) into
profiles/r02_* and refresh the c5 / c2 entries of profiles/mttkrp_traffic.json (ROOT MTTKRP DRAM
bytes per call; c3's first-generation kernel is unchanged since its round-2 capture, whose
tiled-tree accounting stays)."""
import collections, csv, io, json, os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G, P = f'{R}/gpurun_out', f'{R}/profiles'
pre = sys.argv[1] if len(sys.argv) > 1 else 'fin'


def last_json(path):
    lines = [l for l in open(path).read().strip().splitlines() if l.startswith('{')]
    return json.loads(lines[-1])


for c in ['c5', 'c3', 'c2']:
    f = f'{G}/{pre}_bench_{c}.json'
    if os.path.exists(f):
        json.dump(last_json(f), open(f'{P}/r02_bench_{c}.json', 'w'))
f = f'{G}/{pre}_reference_c5.json'
if os.path.exists(f):
    json.dump(last_json(f), open(f'{P}/r02_reference_c5.json', 'w'))
for src, dst in [(f'{pre}_c5_launches.csv', 'r02_c5_launches.csv'),
                 (f'{pre}_gpu_pytest.log', 'r02_gpu_pytest.log'), (f'{pre}_smoke.log', 'r02_smoke.log')]:
    if os.path.exists(f'{G}/{src}'):
        open(f'{P}/{dst}', 'w').write(open(f'{G}/{src}').read())
rep = f'{G}/{pre}_root2_c5.ncu-rep'
if os.path.exists(rep):
    for page, dst in [('raw', 'r02_root2_c5_ncu_raw.csv'), ('source', 'r02_root2_c5_ncu_source.csv')]:
        out = subprocess.run(['ncu', '-i', rep, '--page', page, '--csv'], capture_output=True,
                             text=True).stdout
        open(f'{P}/{dst}', 'w').write(out)


def num(x):
    return float(x.replace(',', ''))


traffic = json.load(open(f'{P}/mttkrp_traffic.json'))
for c in ['c5', 'c3', 'c2']:
    f = f'{G}/{pre}_traffic_{c}.csv'
    if not os.path.exists(f):
        continue
    txt = open(f).read()
    i = txt.index('"ID"')
    open(f'{P}/r02_traffic_{c}.csv', 'w').write(txt[i:])
    if c == 'c3':
        continue
    rr = list(csv.reader(io.StringIO(txt[i:])))
    hh = rr[0]
    per = collections.defaultdict(dict)
    for r in rr[1:]:
        if len(r) == len(hh):
            per[r[hh.index('ID')]][r[hh.index('Metric Name')]] = (
                num(r[hh.index('Metric Value')]), r[hh.index('Metric Unit')])
    sc = lambda v: v[0] * {'Mbyte': 1e6, 'Gbyte': 1e9, 'Kbyte': 1e3, 'byte': 1}.get(v[1], 1)
    ms = lambda v: v[0] * {'msecond': 1.0, 'ms': 1.0, 'usecond': 1e-3, 'us': 1e-3, 'nsecond': 1e-6, 'ns': 1e-6}.get(v[1], 1)
    tot = [sc(m['dram__bytes_read.sum']) + sc(m['dram__bytes_write.sum']) for m in per.values()]
    t = [ms(m['gpu__time_duration.sum']) for m in per.values()]
    hit = sum(m['lts__t_sector_hit_rate.pct'][0] * x for m, x in zip(per.values(), t)) / sum(t)
    l1 = sum(m['l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'][0] * x
             for m, x in zip(per.values(), t)) / sum(t)
    traffic[f'{c}:G1'] = {
        "dram_bytes_per_launch": sum(tot) / len(tot), "l2_hit_rate_pct": hit,
        "l1tex_wavefront_pct": l1, "ncu_ms_per_launch": sum(t) / len(t),
        "source": f"round 2 final: profiles/r02_traffic_{c}.csv (ncu --metrics ... -k regex:mttkrp "
                  f"-s 4 -c 8, bench.py --config {c} --iters 3)"}
json.dump(traffic, open(f'{P}/mttkrp_traffic.json', 'w'), indent=1)
print(json.dumps({k: v for k, v in traffic.items() if k != '_source'}, indent=1))
