"""Per-pass device timeline of one persistent solve (perf-iteration aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N

kind = sys.argv[1] if len(sys.argv) > 1 else "weak"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**8
if kind in ("weak", "corr", "unc", "jac"):
    fam = {"weak": "cqk-weakly-correlated", "corr": "cqk-correlated", "unc": "cqk-uncorrelated",
           "jac": "cqk-weakly-correlated"}[kind]
    d, a, b, l, u, r = P.instances.gen_cqk_arrays(fam, n, 1)
    inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    f = (lambda: P.jacobi_solve(inst)) if kind == "jac" else (lambda: P.solve_cqk(inst))
    B = {0: 40, 1: 40, 2: 40}
    fin = 48
else:
    fam = "simplex-u01" if kind.endswith("u01") else "simplex-n01"
    y = torch.from_numpy(P.gen_simplex_y(fam, n, 1)).cuda()
    start = os.environ.get("CQK_START", "auto")
    f = ((lambda: P.newton_project_simplex(y, 1.0, start=start)) if kind.startswith("spx")
         else (lambda: P.simplex.project_l1_outcome(y, 1.0, start=start)))
    B = {0: 8, 1: 8, 6: 8}
    fin = 16
for _ in range(3):
    out = f()
torch.cuda.synchronize()
h = N.handle()
tl = h.timeline(64)
t0 = tl[0, 3]
prev = t0
prev_rel = t0
rows = []
last = 0
for k in range(1, len(tl)):
    ph, el, comp, t = (int(v) for v in tl[k][:4])
    t_all, t_rel, t_arr1, t_wake1, last_cta, t_last = (int(v) for v in tl[k][4:10])
    t_start, t_cons, t_red, t_prod, t_lastw, t_pre = (int(v) for v in tl[k][10:16])
    m_start, m_load, m_shfl, m_fold = (int(v) for v in tl[k][16:20])
    if t == 0 or t < prev:
        break
    dt = (t - prev) / 1e3
    by = el * B.get(ph, 40)
    rows.append({"epoch": k, "phase": ph, "elems": el, "compact": comp, "us": round(dt, 1),
                 "GBps": round(by / dt / 1e3, 0) if dt > 0 else None,
                 # breakdown (us): previous release -> CTA1 woke -> CTA1 arrived;
                 # all arrived -> decision start -> released
                 "wake1": round((t_wake1 - prev_rel) / 1e3, 2) if prev_rel and t_wake1 else None,
                 "arrive1": round((t_arr1 - prev_rel) / 1e3, 2) if prev_rel and t_arr1 else None,
                 "all_arrived": round((t_all - prev_rel) / 1e3, 2) if prev_rel and t_all else None,
                 "reduced": round((t - t_all) / 1e3, 2) if t_all else None,
                 "released": round((t_rel - t) / 1e3, 2) if t_rel else None,
                 "last_cta": last_cta,
                 "last_arrived": round((t_last - prev_rel) / 1e3, 2) if t_last else None,
                 # CTA 1 (TMA kernels): pass start / consumers done / reduced / producer done
                 "c1_start": round((t_start - prev_rel) / 1e3, 2) if t_start and prev_rel else None,
                 "c1_cons": round((t_cons - prev_rel) / 1e3, 2) if t_cons and prev_rel else None,
                 "c1_red": round((t_red - prev_rel) / 1e3, 2) if t_red and prev_rel else None,
                 "c1_prod": round((t_prod - prev_rel) / 1e3, 2) if t_prod and prev_rel else None,
                 "c1_lastwarp": round((t_lastw - prev_rel) / 1e3, 2) if t_lastw and prev_rel else None,
                 "c1_last_tid": t_lastw & 511,
                 "m_start": round((m_start - t_all) / 1e3, 2) if m_start and t_all else None,
                 "m_load": round((m_load - t_all) / 1e3, 2) if m_load and t_all else None,
                 "m_shfl": round((m_shfl - t_all) / 1e3, 2) if m_shfl and t_all else None,
                 "m_fold": round((m_fold - t_all) / 1e3, 2) if m_fold and t_all else None,
                 "c1_pre": round((t_pre - prev_rel) / 1e3, 2) if t_pre and prev_rel else None})
    prev_rel = t_rel
    prev = t
    last = t
# the final pass's row (the epoch after the last decision): CTA 0 / CTA 1 start, end
if True:
    rel = int(max(tl[1:, 5]))  # the last release
    fr = [r_ for r_ in tl[1:] if r_[11]]
    if fr:
        fr = fr[-1]
        for k_, r_ in enumerate(tl[1:], 1):
            if kind not in ("weak", "corr", "unc", "jac") and r_[15] and r_[14]:
                print(json.dumps({"tail_entry_row": k_, "decided_to_drained_us": round((int(r_[14]) - int(r_[3])) / 1e3, 2),
                                  "gather_us": round((int(r_[15]) - int(r_[14])) / 1e3, 2),
                                  "first_iter_us": round((int(tl[k_ + 1][3]) - int(r_[15])) / 1e3, 2)}))
        print(json.dumps({"final_row": {"m_start": round((int(fr[10]) - rel) / 1e3, 2),
                                        "m_end": round((int(fr[11]) - rel) / 1e3, 2),
                                        "c1_start": round((int(fr[12]) - rel) / 1e3, 2) if fr[12] else None,
                                        "c1_end": round((int(fr[13]) - rel) / 1e3, 2) if fr[13] else None,
                                        "last_cta_end": round((int(fr[15]) - rel) / 1e3, 2) if fr[15] else None}}))
tot_ms = out.stats["device_ms"]
final_us = tot_ms * 1e3 - (last - t0) / 1e3
rows.append({"phase": "final(+launch)", "elems": n, "us": round(final_us, 1),
             "GBps": round(n * fin / final_us / 1e3, 0)})
print(json.dumps({"kind": kind, "n": n, "kernel_ms": tot_ms, "evals": out.phi_evals,
                  "bytes_model": out.stats["bytes_model"]}))
for r_ in rows:
    print(json.dumps(r_))
