"""Generate the golden vectors for the 2D tree SWDFT path FROM THE REFERENCE ITSELF.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports swdft (the unmodified reference at /root/reference/pkg/src) and
records its outputs for seeded inputs:
  * SPEC.md known-answer tests, full values;
  * the acceptance-1/2 sweep: 50 seeded complex arrays up to
    16x16, all windows {1,2,4,8}^2 -> SHA-256 of the complex128 output bytes;
  * config 1 (BASELINE.json configs[0]) full output SHA-256 + sample windows;
  * sampled windows and small strips of configs 2-5 (values / SHA-256),
    computed by running the reference on the window's (or strip's) own input
    sub-array, which is bitwise identical to the full run;
  * OpCounter totals / per-position counts (bench.OpCounter, tree2d.py:90-92,115-118);
  * budget accounting (core.output_bytes, acceptance 5) and twiddle tables.
Inputs are NOT stored (they are regenerated from their seeds; their SHA-256 is
stored so a mismatch is detected).  Nothing here runs on the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF = os.environ.get("SWDFT_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from swdft import bench as ref_bench  # noqa: E402
from swdft import core as ref_core  # noqa: E402
from swdft import tree2d as ref_tree2d  # noqa: E402

from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_run(x, m0, m1, normalization="none"):
    spec = ref_core.WindowSpec((m0, m1), normalization)
    return ref_tree2d.tree_swdft_2d(x, spec, budget=1 << 62).values


def acc_input(case: int):
    rng = np.random.default_rng(1000 + case)
    N0 = int(rng.integers(8, 17))
    N1 = int(rng.integers(8, 17))
    x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
    return x


def sample_positions(cfg, count: int, seed: int):
    P0, P1 = cfg.P0, cfg.P1
    pts = [(0, 0), (0, P1 - 1), (P0 - 1, 0), (P0 - 1, P1 - 1), (P0 // 2, P1 // 2),
           (0, P1 // 2), (P0 // 2, 0)]
    rng = np.random.default_rng(seed)
    while len(pts) < count:
        pts.append((int(rng.integers(0, P0)), int(rng.integers(0, P1))))
    return pts


def main():
    arrays = {}
    meta = {"reference": REF, "numpy": np.__version__}

    # --- SPEC KATs
    kat = {}
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    arrays["kat1_out"] = ref_run(x, 1, 1)
    kat["kat1"] = {"x": x.tolist(), "m": [1, 1]}
    x = np.ones((8, 8))
    arrays["kat2_out"] = ref_run(x, 2, 2)
    kat["kat2"] = {"shape": [8, 8], "m": [2, 2]}
    rng = np.random.default_rng(77)
    x = rng.standard_normal((6, 8)) + 1j * rng.standard_normal((6, 8))
    arrays["kat6_x"] = x
    arrays["kat6_out"] = ref_run(x, 1, 2)
    x = rng.standard_normal((12, 10))
    arrays["norm_x"] = x
    for mode in ("unitary", "paper-2d"):
        arrays[f"norm_{mode}_out"] = ref_run(x, 2, 1, mode)
    meta["kat"] = kat

    # --- acceptance 1/2 sweep (hashes)
    acc = []
    for case in range(50):
        x = acc_input(case)
        for m0 in range(4):
            for m1 in range(4):
                if (1 << m0) > x.shape[0] or (1 << m1) > x.shape[1]:
                    continue
                out = ref_run(x, m0, m1)
                acc.append({"case": case, "m0": m0, "m1": m1, "in_sha": sha(x), "sha": sha(out),
                            "shape": list(out.shape)})
    meta["acc"] = acc

    # --- configs
    cfgs = {}
    for name, cfg in CONFIGS.items():
        x = cfg.generate()
        entry = {"in_sha": sha(x)}
        if name == "c1":
            out = ref_run(x, cfg.m0, cfg.m1)
            entry["full_sha"] = sha(out)
            entry["full_shape"] = list(out.shape)
            arrays["c1_full_out_rows0_4"] = out[:4]
        pts = sample_positions(cfg, 12 if name != "c5" else 8, seed=int(name[1:]) * 31 + 5)
        wins = []
        for (p0, p1) in pts:
            sub = x[p0:p0 + cfg.n0, p1:p1 + cfg.n1]
            wins.append(ref_run(sub, cfg.m0, cfg.m1)[0, 0])
        arrays[f"{name}_win_pos"] = np.array(pts, dtype=np.int64)
        arrays[f"{name}_win_out"] = np.stack(wins)
        # small strips: window rows [a, a+2) x window columns [b, b+W)
        W = 48 if name != "c5" else 24
        strips = []
        for (a, b) in [(0, 0), (cfg.P0 // 2, cfg.P1 // 3), (cfg.P0 - 2, cfg.P1 - W)]:
            sub = x[a:a + 2 + cfg.n0 - 1, b:b + W + cfg.n1 - 1]
            out = ref_run(sub, cfg.m0, cfg.m1)
            strips.append({"p0": a, "p1": b, "rows": 2, "cols": W, "sha": sha(out)})
        entry["strips"] = strips
        cfgs[name] = entry
        print(name, "done", flush=True)
    meta["configs"] = cfgs

    # --- op counter (both loop orders)
    ops = []
    for (N0, N1, m0, m1) in [(20, 17, 2, 3), (33, 40, 3, 1), (9, 9, 0, 2), (12, 12, 3, 3), (5, 7, 0, 0)]:
        x = np.random.default_rng(N0 * 100 + N1).standard_normal((N0, N1))
        spec = ref_core.WindowSpec((m0, m1))
        rec = {"N0": N0, "N1": N1, "m0": m0, "m1": m1}
        for order in ("levels-outer", "trees-outer"):
            c = ref_bench.OpCounter((N0, N1))
            ref_tree2d.tree_swdft_2d(x, spec, loop_order=order, counter=c)
            rec[order] = {"total": int(c.total), "pos_sha": sha(c.position_ops),
                          "pos_sum": int(c.position_ops.sum())}
        rec["predict_ops"] = int(ref_bench.predict_ops("tree", (N0, N1), (1 << m0, 1 << m1)))
        ops.append(rec)
    meta["opcount"] = ops
    per_window = {}
    for n in (2, 4, 8, 16, 32):
        x = np.ones((2 * n, 2 * n))
        c = ref_bench.OpCounter((2 * n, 2 * n))
        ref_tree2d.tree_swdft_2d(x, ref_core.WindowSpec.from_sizes((n, n)), counter=c)
        per_window[str(n)] = int(c.position_ops[-1, -1])
    meta["ops_per_interior_window"] = per_window

    # --- budget accounting
    spec32 = ref_core.WindowSpec.from_sizes((32, 32))
    meta["budget"] = {
        "paper_output_bytes": ref_core.output_bytes((431, 431), spec32),
        "paper_lattice_bytes": ref_core.lattice_bytes((431, 431), spec32),
    }
    try:
        ref_tree2d.tree_swdft_2d(np.ones((8, 8)), ref_core.WindowSpec((1, 1)), budget=10)
    except ref_core.BudgetError as e:
        meta["budget"]["error"] = {"required": e.required_bytes, "budget": e.budget_bytes,
                                   "msg": str(e)}

    # --- next rows: container bytes, 1D tree, 1x1 stream, verify, bench ops
    from swdft import cli as ref_cli  # noqa: E402
    from swdft import container as ref_container  # noqa: E402
    from swdft import tree1d as ref_tree1d  # noqa: E402
    import tempfile

    nxt = {}
    with tempfile.TemporaryDirectory() as td:
        x = np.random.default_rng(21).standard_normal((12, 9))
        out = ref_tree2d.tree_swdft_2d(x, ref_core.WindowSpec((2, 1), "unitary"))
        pth = os.path.join(td, "c.swdf")
        ref_container.write_swdf(pth, out.values, normalization=out.normalization)
        nxt["swdf_unitary_12x9_w4x2"] = hashlib.sha256(open(pth, "rb").read()).hexdigest()
        ref_container.write_swdf(pth, x)
        nxt["swdf_real_12x9"] = hashlib.sha256(open(pth, "rb").read()).hexdigest()
        # cmd_verify on a CSV input, normal and --corrupt (exit code + printed line)
        csvp = os.path.join(td, "x.csv")
        np.savetxt(csvp, x, delimiter=",")
        import contextlib
        import io as _io
        res = {}
        for flag in ([], ["--corrupt"]):
            buf = _io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = ref_cli.main(["verify", "--input", csvp, "--window", "4x2"] + flag)
            res["corrupt" if flag else "plain"] = {"rc": rc, "line": buf.getvalue().strip()}
        nxt["verify"] = res
        # cmd_transform: CSV in, SWDF out (file bytes)
        outp = os.path.join(td, "t.swdf")
        with contextlib.redirect_stdout(_io.StringIO()):
            rc = ref_cli.main(["transform", "--input", csvp, "--output", outp, "--window", "4x2",
                               "--normalization", "paper-2d"])
        nxt["transform"] = {"rc": rc, "sha": hashlib.sha256(open(outp, "rb").read()).hexdigest()}
    sigs = []
    for i, (N, m) in enumerate([(40, 3), (17, 4), (9, 0), (64, 6)]):
        s1 = np.random.default_rng(300 + i).standard_normal(N) + 1j * np.random.default_rng(400 + i).standard_normal(N)
        c = ref_bench.OpCounter((N,))
        v = ref_tree1d.tree_swdft_1d(s1, ref_core.WindowSpec((m,)), counter=c).values
        sigs.append({"N": N, "m": m, "seed_re": 300 + i, "seed_im": 400 + i, "sha": sha(v),
                     "total": int(c.total), "pos_sha": sha(c.position_ops)})
    nxt["tree1d"] = sigs
    # the reference stream works for 1x1 windows only (App. A #11)
    xs = np.random.default_rng(55).standard_normal((7, 6))
    st = ref_tree2d.SlidingRowStream2D(ref_core.WindowSpec((0, 0)), 6)
    slabs = [st.push_row(r) for r in xs]
    nxt["stream_1x1_sha"] = sha(np.stack(slabs))
    # the reference's 1D sample-push stream (it works): emitted vectors + per-push ops
    sig = np.random.default_rng(57).standard_normal(40) + 1j * np.random.default_rng(58).standard_normal(40)
    c1 = ref_bench.OpCounter((40,))
    s1 = ref_tree1d.SlidingStream1D(ref_core.WindowSpec((3,), "paper-1d"), counter=c1)
    outs, ops1 = [], []
    for v in sig:
        r = s1.push(v)
        ops1.append(s1.ops_last_push)
        if r is not None:
            outs.append(r)
    nxt["stream1d"] = {"sha": sha(np.stack(outs)), "ops": ops1, "total": int(c1.total),
                       "pos_sha": sha(c1.position_ops)}
    nxt["fig4_predict_ops"] = {f"{w}": {a: int(ref_bench.predict_ops(a, (100, 100), (w, w)))
                                        for a in ("tree", "fft", "naive")}
                               for w in (4, 8, 16, 32, 64)}
    # kD (treekd.tree_swdft_kd), SPEC acceptance 6 shapes plus a larger 3D case
    from swdft import treekd as ref_treekd  # noqa: E402
    kd = []
    for i, (shape, m, mode) in enumerate([((6, 6, 6), (1, 1, 1), "none"), ((6, 6, 6), (2, 1, 1), "none"),
                                          ((4, 4, 4, 4), (1, 1, 1, 1), "none"),
                                          ((12, 10, 9), (2, 1, 2), "unitary"), ((9, 8, 7), (3, 0, 2), "none")]):
        rng = np.random.default_rng(600 + i)
        xk = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        c = ref_bench.OpCounter(shape)
        v = ref_treekd.tree_swdft_kd(xk, ref_core.WindowSpec(m, mode), counter=c).values
        kd.append({"shape": list(shape), "m": list(m), "mode": mode, "seed": 600 + i, "sha": sha(v),
                   "total": int(c.total), "pos_sha": sha(c.position_ops)})
    nxt["treekd"] = kd
    meta["next"] = nxt

    # --- twiddles
    meta["twiddles"] = {str(1 << k): sha(ref_core.make_twiddles(1 << k)) for k in range(13)}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
