"""Debug helper: E_val components (device chunk states vs oracle) for one workload."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import paper_2605_20868_b200 as ck
import oracle
from oracle.step import make_workload, OraclePolicy, phase1

kw = dict(kind="gaussian", n_tokens=520, query_heads=8, kv_heads=2, steps=1, seed=0)
cfg = ck.WorkloadConfig(head_dim=128, ingest_binary16=True, **kw)
wl = ck.generate_workload(cfg)
dec = ck.CertifiedDecoder(wl.cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4)
res = dec.step(torch.from_numpy(wl.queries[0].reshape(2, 4, 128)).cuda())
ow = make_workload(head_dim=128, ingest_binary16=True, narrow=True, **kw)
C = dec.st.n_chunks
print("n_work", dec.n_work.cpu().tolist(), "C", C)
for h in range(8):
    u, j = divmod(h, 4)
    kv = ow["caches"][u]
    r = oracle.decode_step(ow["queries"][0, h], kv, OraclePolicy(exploration_rate=0.0))
    cs = dec.chunk_state[u, :, j].cpu().numpy()
    valid = cs[:, 0] != -np.inf
    eF = sum(cs[k, 4:6].view(np.float64)[0] for k in range(C) if valid[k])
    sF = sum(cs[k, 6:8].view(np.float64)[0] for k in range(C) if valid[k])
    lm2 = dec.lm2[u, j, :kv.num_blocks].double().cpu().numpy()
    hsb = dec.head_state[u, j].cpu().numpy()
    lse = hsb[0:2].view(np.float64)[0]
    eta = kv.etas()
    vp = set(r["value_promotions"].tolist())
    F = r["promoted"].tolist()
    eF_ref = sum(np.exp(r["log_mass_p2"][b] - lse) * eta[b] for b in F if b not in vp)
    sF_ref = sum(np.exp(r["log_mass_p2"][b] - lse) for b in F)
    print(f"h{h} e_val dev {res.cert[u,j]['e_val']:.6f} ref {r['e_val']:.6f} eF {eF:.6f}/{eF_ref:.6f} sF {sF:.6f}/{sF_ref:.6f} "
          f"lm2 err {np.abs(lm2[F]-r['log_mass_p2'][F]).max():.2e} V dev {res.value_promotions(u,j).tolist()} ref {sorted(vp)} chunks {valid.sum()}")
