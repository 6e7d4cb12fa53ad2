"""Shared test helpers: golden-fixture loading and conversion to oracle / product forms."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def _s(v) -> str:
    return str(np.asarray(v).item() if np.asarray(v).ndim == 0 else v)


def oracle_bank(z: dict, prefix: str) -> dict:
    kind = _s(z[f"{prefix}.kind"])
    gs = int(z[f"{prefix}.group_size"])
    ch = int(z[f"{prefix}.channels"])
    if kind in ("explicit", "mixed"):
        filters = [("explicit", t) for t in z[f"{prefix}.taps"]]
    elif kind == "regularized":
        filters = [("regularized", t, float(r), float(b)) for t, r, b in
                   zip(z[f"{prefix}.taps_hat"], z[f"{prefix}.rate"], z[f"{prefix}.base"])]
    else:
        length = int(z[f"{prefix}.length"])
        filters = [("implicit", r, p, length) for r, p in zip(z[f"{prefix}.residues"], z[f"{prefix}.poles"])]
    return {"channels": ch, "group_size": gs, "filters": filters}


def oracle_cfg(z: dict, prefix: str) -> dict:
    cfg = {"variant": _s(z[f"{prefix}.variant"]), "width": int(z[f"{prefix}.width"]),
           "block_size": int(z[f"{prefix}.block_size"]), "backend": _s(z[f"{prefix}.backend"])}
    for name in ("w_q", "w_k", "w_v", "w_out"):
        # factored projections (hyena.py:48-65) are stored as .left / .right next to the dense
        cfg[name] = ((z[f"{prefix}.{name}.left"], z[f"{prefix}.{name}.right"])
                     if f"{prefix}.{name}.left" in z else z[f"{prefix}.{name}"])
    for name in ("q_feat", "k_feat", "v_feat", "inner"):
        cfg[name] = oracle_bank(z, f"{prefix}.{name}")
    return cfg


def product_bank(z: dict, prefix: str):
    from paper_2503_01868_b200 import ExplicitFilter, GroupSpec, ImplicitFilter, RegularizedFilter
    b = oracle_bank(z, prefix)
    filters = []
    for f in b["filters"]:
        if f[0] == "explicit":
            filters.append(ExplicitFilter(f[1]))
        elif f[0] == "regularized":
            filters.append(RegularizedFilter(f[1], f[2], f[3]))
        else:
            filters.append(ImplicitFilter(f[1], f[2], f[3]))
    return GroupSpec(b["channels"], b["group_size"], tuple(filters))


def product_cfg(z: dict, prefix: str):
    from paper_2503_01868_b200 import HyenaConfig
    o = oracle_cfg(z, prefix)
    return HyenaConfig(
        variant=o["variant"], width=o["width"],
        w_q=o["w_q"], w_k=o["w_k"], w_v=o["w_v"], w_out=o["w_out"],
        q_feat=product_bank(z, f"{prefix}.q_feat"), k_feat=product_bank(z, f"{prefix}.k_feat"),
        v_feat=product_bank(z, f"{prefix}.v_feat"), inner=product_bank(z, f"{prefix}.inner"),
        block_size=o["block_size"], backend=o["backend"])


def explicit_bank_from_taps(taps: np.ndarray, gs: int) -> dict:
    taps = np.atleast_2d(np.asarray(taps, dtype=np.float64))
    return {"channels": taps.shape[0] * gs, "group_size": gs,
            "filters": [("explicit", t) for t in taps]}


def product_groups_from_taps(taps: np.ndarray, gs: int):
    from paper_2503_01868_b200 import ExplicitFilter, GroupSpec
    taps = np.atleast_2d(np.asarray(taps, dtype=np.float64))
    return GroupSpec(taps.shape[0] * gs, gs, tuple(ExplicitFilter(t) for t in taps))


def grads_from_golden(z: dict, prefix: str) -> dict:
    """The flat arrays written by make_golden.grads_arrays, back in the oracle's grads form."""
    out = {"dx": z[f"{prefix}.dx"], "filters": {}}
    for name in ("dw_q", "dw_k", "dw_v", "dw_out"):
        out[name] = ((z[f"{prefix}.{name}.left"], z[f"{prefix}.{name}.right"])
                     if f"{prefix}.{name}.left" in z else z[f"{prefix}.{name}"])
    for key in z:
        if key.startswith(f"{prefix}.f."):
            role, leaf = key[len(prefix) + 3:].split(".")
            out["filters"].setdefault(role, {})[leaf] = z[key]
    return out


def stack_filter_grads(per_group: list) -> dict:
    """[{leaf: grad} per group] -> {leaf: (n_groups, ...)}."""
    return {leaf: np.stack([d[leaf] for d in per_group]) for leaf in per_group[0]}
