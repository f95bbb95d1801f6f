"""Time the regular SLP pair-block kernel variants (H2B_SLP_VARIANT) on config 1."""
import os, sys, subprocess, json
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
from paper_2001_05523_b200.containers import near_slp_jobs, torch, bench
    from paper_2001_05523_b200 import kernels, clustering as C, spaces
    from paper_2001_05523_b200.containers import AssemblyContext, near_layout
    from paper_2001_05523_b200.mesh import sphere_mesh
    m = sphere_mesh(6); ctx = AssemblyContext(m)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 64)
    bt = C.BlockTree(tree, tree, 2.0); lay = near_layout(bt)
    Dn = torch.zeros(lay.total, dtype=torch.float64, device="cuda"); nu = bt.near_uids
    jobs = near_slp_jobs(bt)
    sj = kernels.SlpJobs(ctx.dmesh, 3, jobs, tree.perm.astype(np.int32), tree.perm.astype(np.int32))
    tab = kernels.SingularTable(ctx.dmesh, "slp", 4)
    for _ in range(2): sj.run(tab, Dn)
    t = bench.ev_time(torch, lambda: sj.run(tab, Dn), 10)
    ref = np.load("/tmp/nf_ref.npy") if os.path.exists("/tmp/nf_ref.npy") else None
    h = Dn.cpu().numpy()
    if ref is None: np.save("/tmp/nf_ref.npy", h); err = 0.0
    else: err = float(np.abs(h - ref).max() / np.abs(ref).max())
    fl = (lay.entries - ctx.dmesh.touch().n_pairs) * 81 * 12
    print(json.dumps({"ms": t * 1e3, "tflops": fl / t / 1e12, "err_vs_v0": err}))
else:
    for v in sys.argv[1:] or ["0", "1", "2", "3", "4", "5"]:
        env = dict(os.environ, H2B_SLP_VARIANT=v)
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print("variant", v, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:])
