import json, sys, time
sys.path.insert(0, '.')
from paper_2011_03602_b200.evaluator import B200Evaluator
g = json.load(open('tests/golden/himeno_M_red.json'))
ev = B200Evaluator(g['spec'], devices=[0])
ev.app_for(g['doc'])
for _ in range(2):
    r = ev.measure_payloads(g['doc'], [g['patterns']['100100100']])[0]
print(r['time_s'], r['h2d_bytes'], r['d2h_bytes'], r['launches'])
