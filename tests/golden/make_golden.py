"""Generate golden fixtures for the hot path FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

It alias-imports the reference package as ``harpia_ref`` and
records, for seeded small inputs, the reference outputs of every hot-path
operator (filters.py / morphology.py / registry.py), the chunk plans of
plan_chunks, and the Gaussian taps.  The fixtures travel with the repo; the
GPU box never needs /root/reference.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def load_ref(path: str):
    spec = importlib.util.spec_from_file_location(
        "harpia_ref", f"{path}/harpia/__init__.py", submodule_search_locations=[f"{path}/harpia"])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["harpia_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def volumes(rng):
    """Seeded inputs: ragged shapes, degenerate axes, all supported dtypes."""
    out = {}
    out["f32_a"] = (rng.random((12, 14, 16)) * 1000).astype(np.float32)
    out["f32_unit"] = rng.random((9, 20, 11), dtype=np.float32)
    out["f32_thin"] = rng.random((1, 7, 33), dtype=np.float32)
    out["f32_col"] = rng.random((19, 1, 1), dtype=np.float32)
    out["u8_a"] = rng.integers(0, 256, size=(10, 13, 17), dtype=np.uint8)
    out["u16_a"] = rng.integers(0, 65536, size=(8, 9, 21), dtype=np.uint16)
    out["bin_a"] = (rng.random((11, 12, 13)) < 0.5).astype(np.uint8)
    out["f32_neg"] = (rng.standard_normal((7, 18, 10)) * 50).astype(np.float32)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    ref = load_ref(args.ref)
    F, M, R = ref.filters, ref.morphology, ref.registry
    rng = np.random.default_rng(20251117)
    vols = volumes(rng)
    arrays = {f"in__{k}": v for k, v in vols.items()}
    cases = []

    def add(name, op, params, vol, out):
        key = f"out__{name}"
        arrays[key] = out
        cases.append({"name": name, "op": op, "params": params, "input": f"in__{vol}",
                      "output": key})

    for vol in ("f32_a", "f32_unit", "f32_thin", "f32_col", "u8_a", "u16_a", "f32_neg"):
        for sigma in (0.5, 1.0, 2.0):
            add(f"gaussian_{vol}_{sigma}", "gaussian", {"sigma": sigma}, vol,
                F.gaussian(vols[vol], sigma))
        for r in (1, 2):
            add(f"mean_{vol}_{r}", "mean", {"radius": r}, vol, F.mean(vols[vol], r))
            add(f"median_{vol}_{r}", "median", {"radius": r}, vol, F.median(vols[vol], r))
        add(f"unsharp_{vol}", "unsharp", {"sigma": 1.0, "amount": 1.5}, vol,
            F.unsharp(vols[vol], 1.0, 1.5))
        h = F.hessian(vols[vol], 1.5)
        add(f"log_{vol}", "log", {"sigma": 1.5}, vol, (h["xx"] + h["yy"]) + h["zz"])
    add("median_u8_r3", "median", {"radius": 3}, "u8_a", F.median(vols["u8_a"], 3))
    # the next local map ops on the same machinery
    T = ref.threshold
    for vol in ("f32_a", "f32_neg", "u8_a", "f32_col", "f32_thin"):
        for comp in F.HESSIAN_COMPONENTS:
            add(f"hessian_{comp}_{vol}", f"hessian_{comp}", {"sigma": 1.5}, vol,
                F.hessian_component(vols[vol], 1.5, comp))
    for vol in ("f32_a", "f32_unit", "f32_thin", "f32_col", "u8_a", "u16_a", "f32_neg"):
        add(f"sobel_{vol}", "sobel", {}, vol, F.sobel(vols[vol]))
        add(f"prewitt_{vol}", "prewitt", {}, vol, F.prewitt(vols[vol]))
    for vol in ("f32_a", "f32_thin", "f32_col", "u8_a", "u16_a", "bin_a", "f32_neg"):
        add(f"lbp2d_{vol}", "lbp2d", {}, vol, F.lbp2d(vols[vol]))
    # connected components (registry.py:337-351): canonical labels
    Q = ref.quantify
    for vol in ("bin_a", "u8_a", "f32_thin", "f32_col"):
        for conn in (6, 26):
            lab, _n = Q.connected_components(vols[vol], conn)
            add(f"cc_{vol}_{conn}", "connected_components", {"connectivity": conn}, vol, lab)
    # label-volume filters (registry.py:355-383)
    rl = np.random.default_rng(77)
    labvol = rl.integers(0, 4, size=(14, 17, 19)).astype(np.uint32)
    labvol[rl.random(labvol.shape) < 0.3] = 0
    arrays["in__lab_a"] = labvol
    holes = (rl.random((13, 16, 18)) < 0.55).astype(np.uint8)
    arrays["in__holes_a"] = holes
    for vol in ("lab_a", "holes_a", "bin_a"):
        src = arrays[f"in__{vol}"]
        for conn in (6, 26):
            add(f"fill_holes_{vol}_{conn}", "fill_holes", {"connectivity": conn}, vol,
                ref.morphology.fill_holes(src, conn).astype(src.dtype))
            for ms in (1, 3, 9):
                add(f"remove_islands_{vol}_{conn}_{ms}", "remove_islands",
                    {"min_size": ms, "connectivity": conn}, vol,
                    ref.morphology.remove_islands(src, ms, conn))
    # exact EDT (registry.py:404-417)
    for vol in ("bin_a", "holes_a", "lab_a"):
        for sp in ((1.0, 1.0, 1.0), (2.0, 0.5, 0.75)):
            add(f"edt_{vol}_{sp[0]}", "edt", {"spacing": list(sp)}, vol,
                Q.edt(arrays[f"in__{vol}"], sp))
    # geodesic reconstruction (registry.py:386-401): marker in params (array key)
    for vol, kind in (("u8_a", "dilation"), ("u16_a", "erosion"), ("f32_unit", "dilation")):
        src = arrays[f"in__{vol}"]
        if kind == "dilation":
            marker = np.where(rl.random(src.shape) < 0.02, src, np.zeros_like(src)).astype(src.dtype)
        else:
            top = np.iinfo(src.dtype).max if src.dtype.kind == "u" else src.max()
            marker = np.where(rl.random(src.shape) < 0.02, src, np.full_like(src, top)).astype(src.dtype)
        arrays[f"marker__{vol}_{kind}"] = marker
        add(f"geodesic_{vol}_{kind}", "geodesic_reconstruct",
            {"marker": f"marker__{vol}_{kind}", "kind": kind}, vol,
            ref.morphology.geodesic_reconstruct(marker, src, kind))
    # global Otsu (registry.py:312-334): binarized output; threshold in meta
    otsu_t = {}
    for vol in ("f32_a", "f32_unit", "u8_a", "u16_a", "f32_neg", "bin_a"):
        for bins in (256, 64):
            try:
                lab, t = T.otsu_binarize(vols[vol], bins)
            except ref.errors.HarpiaError:  # degenerate histogram (e.g. binary u8, 64 bins)
                continue
            add(f"otsu_{vol}_{bins}", "otsu", {"bins": bins}, vol, lab)
            otsu_t[f"otsu_{vol}_{bins}"] = t
    for vol in ("f32_unit", "u8_a", "f32_neg", "f32_col"):
        for mode in F.DIFFUSION_MODES:
            for it, kappa in ((1, 0.4), (3, 25.0)):
                p = {"iterations": it, "kappa": kappa, "dt": 1.0 / 6.0, "mode": mode}
                add(f"diffusion_{mode}_{vol}_{it}", "anisotropic_diffusion", p, vol,
                    F.anisotropic_diffusion(vols[vol], it, kappa, 1.0 / 6.0, mode))
    for vol, ts in (("f32_unit", (0.1, 0.5)), ("u8_a", (127.5, 3.0)), ("u16_a", (30000.25,)),
                    ("f32_neg", (0.0, -12.3))):
        for t in ts:
            add(f"apply_threshold_{vol}_{t}", "apply_threshold", {"t": t}, vol,
                T.apply_threshold(vols[vol], t))
    # local adaptive thresholds (threshold.py:174-217), every kind
    for vol, ws in (("u8_a", (1, 2, 3)), ("u16_a", (1, 2)), ("f32_a", (1, 2)), ("f32_neg", (1, 2)),
                    ("f32_thin", (1,))):
        for kind in T.LOCAL_KINDS:
            for w in ws:
                p = {"kind": kind, "window": w, "k": 0.2 if kind != "niblack" else -0.3, "R": None,
                     "c": 1.5 if kind in ("mean", "median", "gaussian") else 0.0}
                add(f"local_threshold_{kind}_{vol}_{w}", "local_threshold", p, vol,
                    T.local_threshold(vols[vol], kind, w, p["k"], p["R"], p["c"]))
    for vol in ("u8_a", "u16_a", "bin_a", "f32_neg"):
        for se in ("ball:1", "ball:2", "ball:3", "box:1", "cross:2"):
            s = M.StructuringElement.parse(se)
            for op in M.MORPH_OPS:
                add(f"morph_{op}_{vol}_{se}", f"morph_{op}", {"se": se}, vol,
                    M.morph(vols[vol], op, s, 1))
        s = M.StructuringElement.parse("ball:1")
        add(f"morph_open2_{vol}", "morph_open", {"se": "ball:1", "iterations": 2}, vol,
            M.morph(vols[vol], "open", s, 2))
    # asymmetric custom element (non-contiguous rows, off-centre)
    custom = ((0, 0, 0), (1, 0, 2), (0, -1, -1), (-2, 1, 0), (0, 0, -2), (1, 1, 1))
    arrays["se__custom"] = np.array(custom, dtype=np.int32)
    cs = M.StructuringElement(custom)
    add("erode_custom_u16", "erode_offsets", {"offsets": "se__custom"}, "u16_a", M.erode(vols["u16_a"], cs))
    add("dilate_custom_u16", "dilate_offsets", {"offsets": "se__custom"}, "u16_a", M.dilate(vols["u16_a"], cs))

    # chunked registry runs (plan invariance, reference engine) at tight budgets
    from harpia_ref.chunking import MemoryBudget, plan_chunks, OpProfile
    plans = []
    for z, y, x, item, halo, scratch, usable in [
            (100, 1024, 1024, 4, 2, 3, 96 * 2**20), (10, 8, 8, 1, 0, 3, 2**20),
            (37, 5, 7, 4, 3, 8, 16 * 5 * 7 * 4 * 8), (64, 64, 64, 1, 8, 8, 40 * 64 * 64 * 8 + 3)]:
        p = plan_chunks((z, y, x), np.dtype(f"u{item}") if item < 4 else np.float32,
                        OpProfile(halo_z=halo, scratch_factor=scratch), MemoryBudget(usable, 1.0))
        plans.append({"shape": [z, y, x], "itemsize": item, "halo": halo, "scratch": scratch,
                      "usable": usable, "dump": p.dump(), "working_peak": p.working_peak_bytes})
    try:
        plan_chunks((100, 1024, 1024), np.uint32, OpProfile(halo_z=2, scratch_factor=3),
                    MemoryBudget(20 * 2**20, 1.0))
    except ref.errors.BudgetTooSmallError as e:
        plans.append({"error": str(e), "minimum_bytes": e.minimum_bytes})

    # reference profiles for the registered hot-path operators
    profiles = {}
    for name, params in [("gaussian", {"sigma": 2.0}), ("mean", {"radius": 1}),
                         ("median", {"radius": 2}), ("unsharp", {"sigma": 1.0, "amount": 1.5}),
                         ("hessian_xx", {"sigma": 2.0}), ("morph_erode", {"se": "ball:3"}),
                         ("morph_open", {"se": "ball:3", "iterations": 2}),
                         ("identity", {}), ("hessian_xy", {"sigma": 1.5}), ("sobel", {}),
                         ("prewitt", {}), ("apply_threshold", {"t": 0.5}), ("lbp2d", {}),
                         ("anisotropic_diffusion", {"iterations": 3, "kappa": 10.0}),
                         ("local_threshold", {"kind": "sauvola", "window": 2})]:
        op = R.get_operator(name)
        pr = op.profile(R.validate_params(op, params))
        profiles[name] = {"params": params, "halo_z": pr.halo_z, "scratch": pr.scratch_factor,
                          "out_dtype": None if pr.out_dtype is None else str(pr.out_dtype)}
    weights = {str(s): F._gaussian_kernel(s).tolist() for s in (0.3, 0.5, 1.0, 1.2, 1.5, 2.0, 2.5, 3.3, 4.0)}
    balls = {str(r): len(M.StructuringElement.ball(r).offsets) for r in (1, 2, 3, 4)}

    # .vol sidecar text (volume.py:28-75)
    V = ref.volume
    sidecars = []
    for dt, shape, spacing, desc in [("float32", (3, 4, 5), (1.0, 0.5, 0.25), "scan A"),
                                     ("uint16", (64, 2052, 2052), (2.0, 1.0, 1.0), ""),
                                     ("uint8", (1, 1, 1), (0.1, 0.2, 0.3), "tiny: x")]:
        m = V.VolumeMeta(dtype=dt, shape=shape, spacing=spacing, description=desc)
        sidecars.append({"dtype": dt, "shape": list(shape), "spacing": list(spacing),
                         "description": desc, "text": m.to_text()})

    np.savez_compressed(HERE / "golden_arrays.npz", **arrays)
    meta = {"generator": "tests/golden/make_golden.py", "reference": args.ref,
            "cases": cases, "plans": plans, "profiles": profiles, "weights": weights,
            "ball_sizes": balls, "sidecars": sidecars, "otsu_thresholds": otsu_t}
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1))
    print(f"{len(cases)} cases, {sum(a.nbytes for a in arrays.values())} bytes raw")


if __name__ == "__main__":
    main()
