"""Time libh2b.so variants (tools/nf_variants.sh -> _lib/variants/<name>.so)
of the regular SLP pair-block kernel on config 1 (symmetric nearfield jobs).

    python tools/nf_variants.py name1 name2 ...   (GPU box)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import bench
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import kernels, spaces
    from paper_2001_05523_b200.containers import AssemblyContext, near_layout, near_slp_jobs
    from paper_2001_05523_b200.mesh import sphere_mesh

    level = int(os.environ.get("NF_LEVEL", "6"))
    m = sphere_mesh(level)
    ctx = AssemblyContext(m)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 64)
    bt = C.BlockTree(tree, tree, 2.0)
    lay = near_layout(bt)
    Dn = torch.zeros(lay.total, dtype=torch.float64, device="cuda")
    sj = kernels.SlpJobs(ctx.dmesh, 3, near_slp_jobs(bt), tree.perm.astype(np.int32), tree.perm.astype(np.int32))
    tab = kernels.SingularTable(ctx.dmesh, "slp", 4)
    for _ in range(2):
        sj.run(tab, Dn)
    t = bench.ev_time(torch, lambda: sj.run(tab, Dn), 20)
    h = Dn.cpu().numpy()
    ref_path = f"/tmp/nf_ref_{level}.npy"
    if not os.path.exists(ref_path):
        np.save(ref_path, h)
    ref = np.load(ref_path)
    err = float(np.abs(h - ref).max() / np.abs(ref).max())
    t_ev = ctx.dmesh.touch()
    n_touch_eval = int(t_ev.case_counts[0] + (t_ev.case_counts[1] + t_ev.case_counts[2]) // 2)
    fl = (sj.evaluated - n_touch_eval) * 81 * 12
    res = {"level": level, "slp_ms": t * 1e3, "slp_tflops": fl / t / 1e12, "err_vs_first": err}
    if os.environ.get("NF_DLP", "1") == "0":
        print(json.dumps(res))
        sys.exit(0)
    # double layer (P0 rows x P1 columns): the regular pair-block kernel with the vertex scatter
    import ctypes

    from paper_2001_05523_b200 import _lib
    from paper_2001_05523_b200 import device as D
    from paper_2001_05523_b200.containers import _near_blocks

    t1 = C.build_cluster_tree(spaces.DofSpace(spaces.P1, m).support_boxes(), 64)
    btd = C.BlockTree(tree, t1, 2.0)
    layd = near_layout(btd)
    packed = kernels.build_dlp_jobs(m, _near_blocks(btd, layd))
    tabd = kernels.SingularTable(ctx.dmesh, "dlp", 4)
    pp, Qd, lam = ctx.dmesh.panel_points(3)
    tt = {k: D.dev(v) for k, v in packed.items()}
    cj = _lib.DlpJobs(len(packed["jobs"]), tt["jobs"].data_ptr(), tt["row_idx"].data_ptr(), tt["pan_idx"].data_ptr(),
                      tt["inc_ptr"].data_ptr(), tt["inc"].data_ptr(), tt["inc_base"].data_ptr())
    Dd = torch.zeros(layd.total, dtype=torch.float64, device="cuda")

    def dlp():
        _lib.check(_lib.lib().h2b_pair_blocks_dlp(ctypes.byref(ctx.dmesh.c), pp.data_ptr(), lam.data_ptr(), Qd,
                                                  ctypes.byref(cj), ctypes.byref(tabd.touch.c),
                                                  tabd.values_dev.data_ptr(), Dd.data_ptr(), D.stream()))

    dlp()
    td = bench.ev_time(torch, dlp, 10)
    hd = Dd.cpu().numpy()
    if not os.path.exists("/tmp/nf_ref_dlp.npy"):
        np.save("/tmp/nf_ref_dlp.npy", hd)
    rd = np.load("/tmp/nf_ref_dlp.npy")
    pairs = int((packed["jobs"][:, 1] * packed["jobs"][:, 3]).sum())
    res.update(dlp_ms=td * 1e3, dlp_tflops=25.0 * pairs * 81 / td / 1e12,
               dlp_err_vs_first=float(np.abs(hd - rd).max() / np.abs(rd).max()))
    print(json.dumps(res))
else:
    for v in sys.argv[1:]:
        path = os.path.join(ROOT, "paper_2001_05523_b200", "_lib", "variants", v + ".so")
        env = dict(os.environ, H2B_LIB_PATH=path)
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print("variant", v, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:],
              flush=True)
