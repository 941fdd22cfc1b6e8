import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1911_00119_b200 as A
from paper_1911_00119_b200 import abi
space = A.preset_space()
ref = A.reference_latency(space)
t = 0.8 * ref
spec = A.ConstraintSpec(mode=A.Mode.MAXIMIZE_ACCURACY, t_goal=t, e_goal=0.6 * 50.0 * t, pr_threshold=0.95, overhead_budget=0.01 * ref)
envs = [A.realize(A.preset_trace(seed=42 + k, phase_length=30)) for k in range(64)]
for flags in (0, abi.FLAG_NO_FAST):
    r = A.run_batch(space, [spec], envs, "alert", records="f64", trace_dtype=np.float64, flags=flags)
    print("flags", flags, "full", r.agg[:, abi.AGG_FULL_SCAN].sum(), "refined", r.agg[:, abi.AGG_REFINED].sum(), r.decoded()["cand"][:5, 0])
