"""Fixed-work chain launch for ncu (no budget, so replays are identical)."""
import sys, time
sys.path.insert(0, '.')
import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import engine as E
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
chains = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = S.generate_mixed(n, 0); c = S.table_coefficients(); ids = sorted(w.ids())
if len(sys.argv) > 4 and sys.argv[4] == "3class":  # configs[0] mix: code / chat / offline (E2E 1e9 ms)
    code, chat = S.default_slo_classes()
    reqs = [S.Request(r.id, 2 if r.id % 3 == 2 else r.task_class_id, r.input_len, r.true_output_len,
                      r.predicted_output_len) for r in w.requests]
    w = S.Workload(reqs, [code, chat, S.TaskClass(2, "offline", S.SloSpec.e2e(1e9))])
s, i = S.initial_candidates(w, ids, c, 4)
ev = S.evaluate(s, c, w)
pos = {r: k for k, r in enumerate(ids)}
eng = E.Engine(0)
ex, dl = E.build_tables(w, ids, c, 4); eng.set_problem(ex, dl)
eng.prepare([pos[x] for x in s.flatten()], [len(b) for b in s.batches], t0=500.0, tau=0.5, iter=32, seed=0,
            objective_scale=500.0 / ev.g, chains=chains, scale_ladder=(1.0, 10.0, 100.0, 1000.0, 1e4, 1e5))
for r in range(reps):
    eng.launch(); bp, bs, res = eng.fetch()
    print(f"rep {r}: {res.proposals} proposals in {res.kernel_ms:.3f} ms = {res.proposals / res.kernel_ms * 1e3:.3e}/s, g={res.g:.4e} n={res.n_met}")
