import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2110_01470_b200 as psso
fn = psso.make_function("f5", 100)
p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=fn.var_min, var_max=fn.var_max, nsol=1024, nvar=100, niter=1000)
def run():
    return min(psso.run_parallel_batch(p, fn, [0])[0].wall_time_s for _ in range(3))
ref = psso.run_parallel(p, fn, 0)
print("cluster (run_parallel)", ref.wall_time_s * 1e3 / 1000, "us/it", flush=True)
print("cluster batch", run() * 1e3, "us/it", flush=True)
os.environ["PSSO_SWARM_NO_CLUSTER"] = "1"
for gpc in ("16", "8", "4", "2", "1"):
    os.environ["PSSO_SWARM_GPC"] = gpc
    try:
        w = run()
        r = psso.run_parallel_batch(p, fn, [0])[0]
        print("global gpc", gpc, w * 1e3, "us/it", "same" if (r.best_position == ref.best_position).all() else "DIFF", flush=True)
    except Exception as e:
        print("gpc", gpc, "error", e)
