import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2505_23022_b200.sweep import SweepGrid
from paper_2505_23022_b200.batch import BatchEngine, Cell
from oracle import oracle as orc
g = SweepGrid(rates=(2.0,), scales=(0.5,))
t = g.trace_for_rate(2.0)
eng = BatchEngine([t], [Cell(0, g.config, slo_scale=0.5)], outcomes=True, device=torch.device('cuda',0))
eng.launch(); res = eng.results(); out = eng.outcomes(); o = eng.sim_outcomes(0, out)
s = 0.5
ref = orc.run_sim(t.arrival, t.ttft_slo*s, t.tpot_slo*s, t.prompt_len, t.true_out, t.id, t.predicted, orc.make_params(itl=g.config.itl, prefill=g.config.prefill), log_steps=500000, log_ids=3000000)
print({f: (int(res[0][f]), ref['summary'][f]) for f in ('n_steps','request_steps','rejected_ttft','rejected_admission','completed','compliant')})
st = np.asarray(o['status']); rs = ref['status']
d = np.nonzero(st != rs)[0]
print('status diffs', len(d), d[:10])
cs = np.asarray(o['completion_step']); rc = ref['completion_step']
d2 = np.nonzero(cs != rc)[0]
print('completion diffs', len(d2), d2[:10])
for i in list(d[:3]) + list(d2[:3]):
    print(i, 'gpu', st[i], cs[i], 'ref', rs[i], rc[i], 'arr', t.arrival[i], 'ttft', t.ttft_slo[i]*s, 'tpot', t.tpot_slo[i]*s, 'prompt', t.prompt_len[i], 'out', t.true_out[i])
# rejection steps: oracle log (ids per step: admitted, rejected, batch)
L = ref['log']; ids = L['ids']; pos = 0; rej_step = {}
for k in range(len(L['n_admitted'])):
    na, nr, nb = int(L['n_admitted'][k]), int(L['n_rejected'][k]), int(L['n_batch'][k])
    for j in range(nr):
        rej_step[int(ids[pos + na + j]) // 2] = k
    pos += na + nr + nb
idmap = {int(x): i for i, x in enumerate(t.id)}
bad = 0
for rid, k in sorted(rej_step.items(), key=lambda kv: kv[1]):
    i = idmap[rid]
    if st[i] == 1 and cs[i] != k:
        bad += 1
        if bad <= 5:
            print('rej step differs', i, 'gpu', cs[i], 'ref', k, 'arr', t.arrival[i], 'ttft', t.ttft_slo[i] * s, 'prompt', t.prompt_len[i])
print('rejection-step mismatches', bad, 'of', len(rej_step))
