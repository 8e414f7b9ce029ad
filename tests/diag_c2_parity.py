import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
import bench
from parity_common import rel_err
from paper_2508_13716_b200 import api, hostgraph as H
bench.apply_config("c2")
g, ps, caps = bench.build_workload(8)
cfg = H.SimConfig(epochs=3, policy="jaca", staleness_bound=-1, f_dim=bench.F_DIM, L=3)
res = {}
for gemm in ("fp32", "3xtf32"):
    rep = api.train(g, ps, H.unit_profiles(8), caps, cfg, model="gcn", num_classes=40, keep_logits="all", gemm=gemm, keep_params=True)
    res[gemm] = rep
sess = bench.OracleSession(g, ps, caps, -1)
outs = []
for e in range(3):
    sess.e += 1
    plan = sess.planner.step(sess.e, -1)
    outs.append(sess.trainer.step(plan.version))
for gemm, rep in res.items():
    print(gemm, "free:", [f"{rel_err(rep.logits_per_epoch[e], outs[e].logits):.2e}" for e in range(3)],
          "loss:", [f"{abs(rep.losses[e]-outs[e].loss)/abs(outs[e].loss):.2e}" for e in range(3)])
# forced: oracle restarted from the GPU's weights each epoch
from oracle import model_port as omp
for gemm, rep in res.items():
    sess2 = bench.OracleSession(g, ps, caps, -1)
    errs = []
    for e in range(3):
        sess2.e += 1
        plan = sess2.planner.step(sess2.e, -1)
        o = sess2.trainer.step(plan.version, forced_params=rep.params_per_epoch[e])
        errs.append(rel_err(rep.logits_per_epoch[e], o.logits))
    print(gemm, "forced:", [f"{x:.2e}" for x in errs])
# gradient magnitude distribution at epoch 1 (from the fp32 params delta)
p0 = res["fp32"].params_per_epoch[0]; p1 = res["fp32"].params_per_epoch[1]
d = np.concatenate([(b - a).ravel() for a, b in zip(p0, p1)])
print("epoch-1 update |delta|/lr quantiles:", np.quantile(np.abs(d) / 0.01, [0.001, 0.01, 0.1, 0.5]))
