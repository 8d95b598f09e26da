"""Debug helper: compare device intermediates with the oracle for one workload."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
import paper_2605_20868_b200 as ck
import oracle
from oracle.step import make_workload, OraclePolicy, phase1, select_blocks

kind = sys.argv[1] if len(sys.argv) > 1 else "needle"
kw = dict(kind=kind, n_tokens=777, query_heads=8, kv_heads=2, steps=2, seed=2)
pk = dict(k_max=16)
cfg = ck.WorkloadConfig(head_dim=128, ingest_binary16=True, **kw)
wl = ck.generate_workload(cfg)
pol = ck.PolicyConfig(exploration_rate=0.0, **pk)
dec = ck.CertifiedDecoder(wl.cache, pol, n_heads=4)
q = torch.from_numpy(wl.queries[0].reshape(2, 4, 128)).cuda()
res = dec.step(q, dense=False)
ow = make_workload(head_dim=128, ingest_binary16=True, narrow=True, **kw)
for h in range(8):
    u, j = divmod(h, 4)
    kv = ow["caches"][u]
    qq = ow["queries"][0, h]
    r = oracle.decode_step(qq, kv, OraclePolicy(exploration_rate=0.0, **pk))
    nb = kv.num_blocks
    lm1 = dec.lm1[u, j, :nb].double().cpu().numpy()
    p1 = phase1(qq, kv)
    kp = int(res.cert[u, j]["k_star"])
    order = dec.order[u, j, :kp].cpu().numpy()
    lm2 = dec.lm2[u, j, :kp].double().cpu().numpy()
    ref_lm2 = r["log_mass_p2"][order]
    out = res.out[u, j].double().cpu().numpy()
    hs = dec.head_state[u, j].cpu().numpy()
    vl = res.value_promotions(u, j)
    print(f"h{h} lm1 err {np.abs(lm1 - p1['log_mass']).max():.2e} order_eq {sorted(order.tolist()) == r['promoted'].tolist()} "
          f"lm2 err {np.abs(lm2 - ref_lm2).max():.2e} V dev {vl.tolist()} ref {r['value_promotions'].tolist()} "
          f"out err {np.abs(out - r['quant_output']).max() / np.abs(r['quant_output']).max():.2e} "
          f"e_val {res.cert[u,j]['e_val']:.6e} ref {r['e_val']:.6e} delta {res.cert[u,j]['delta_h']:.6e} ref {r['delta_h']:.6e}")

print("---- per-block lm1 error, unit 0 head 1")
u, j = 0, 1
kv = ow["caches"][u]; qq = ow["queries"][0, 1]
p1 = phase1(qq, kv)
lm1 = dec.lm1[u, j, :kv.num_blocks].double().cpu().numpy()
err = lm1 - p1["log_mass"]
np.set_printoptions(precision=2, linewidth=200)
print(err)
print("smax", wl.cache.kscale_max[u, :kv.num_blocks].cpu().numpy())
print("kscale max (oracle)", np.array([kv.kscale[b].astype(np.float32).max() for b in range(kv.num_blocks)]))
print("|z| max", np.array([np.abs(kv.koffset[b]).max() for b in range(kv.num_blocks)]))
