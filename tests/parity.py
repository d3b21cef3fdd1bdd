"""Tolerance gates shared by the GPU parity tests.

Gate A (BASELINE.json north_star, verbatim): on N(0,1) inputs
    out  : max-abs <= 1e-2 and mean-abs <= 1e-3
    dq/dk/dv : max-abs <= 2e-2
    lse  : max-abs <= 1e-3 (fp32 statistics)
Gate B (sharpness): relative L2 <= 1e-2 per tensor, and
elementwise |err| <= atol + 2^-6 |ref| (the bf16 output rounding is 2^-9
relative; P, dS are rounded to bf16 before the second GEMMs).
"""
import inspect
import json
import os

import numpy as np


def _log(kind, stats):
    """With UA_PARITY_LOG=<path>, append the achieved margins of every gate
    (err / bound, <= 1 passes) as JSON lines, tagged with the calling test."""
    path = os.environ.get("UA_PARITY_LOG")
    if not path:
        return
    test = next((f.function for f in inspect.stack() if f.function.startswith("test_")), "?")
    try:
        test = os.environ.get("PYTEST_CURRENT_TEST", test).split(" ")[0]
    except Exception:
        pass
    with open(path, "a") as f:
        f.write(json.dumps(dict(test=test, gate=kind, **stats)) + "\n")


def rel_l2(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30))


def gate_out(x, ref, gate_a=True, absv=None, atol_max=1e-2, atol_mean=1e-3):
    """gate_a: apply the north-star absolute bounds (N(0,1) inputs only).

    Elementwise bound: bf16 has unit roundoff u = 2^-8.  P is rounded to bf16
    before the P.V GEMM, so o_id carries up to u * sum_j P_ij |v_jd| (= absv,
    from the oracle) plus the output rounding u |o_id|; the gate allows twice
    that plus 1e-3 absolute.  Without absv, 2^-6 |ref| is used."""
    err = np.abs(np.asarray(x, np.float64) - ref)
    if gate_a:
        assert err.max() <= atol_max, f"max-abs {err.max():.3e} > {atol_max}"
        assert err.mean() <= atol_mean, f"mean-abs {err.mean():.3e} > {atol_mean}"
    r = rel_l2(x, ref)
    assert r <= 1e-2, f"relL2 {r:.3e}"
    if absv is not None:
        bound = 1e-3 + 2.0 * 2.0 ** -8 * (np.abs(absv) + np.abs(ref))
    else:
        bound = 1e-3 + 2.0 ** -6 * np.abs(ref)
    elt = err - bound
    stats = dict(max=float(err.max()), mean=float(err.mean()), rel_l2=r, elt_margin=float((err / bound).max()),
                 gate_a_max_frac=float(err.max() / atol_max) if gate_a else None,
                 q7_margin=float((err / (1e-3 + 2.0 ** -6 * np.abs(ref))).max()))
    _log("out", stats)
    assert elt.max() <= 0, f"elementwise gate exceeded by {elt.max():.3e}"
    return stats


def gate_lse(x, ref, atol=1e-3):
    err = np.abs(np.asarray(x, np.float64) - ref)
    _log("lse", dict(max=float(err.max()), gate_a_max_frac=float(err.max() / atol)))
    assert err.max() <= atol, f"lse max-abs {err.max():.3e}"
    return float(err.max())


def gate_grad(x, ref, gate_a=True, gabs=None, atol_max=2e-2, rel=1e-2, elt_atol=2e-3):
    """Gradients: relL2 <= 1e-2; elementwise |err| <= elt_atol + 2u(gabs+|ref|)
    with gabs the oracle's error-scale sum (dS or P rounded to bf16 before the
    GEMM, u = 2^-8); Gate A max-abs 2e-2 on N(0,1) inputs."""
    err = np.abs(np.asarray(x, np.float64) - ref)
    r = rel_l2(x, ref)
    assert r <= rel, f"relL2 {r:.3e}"
    scale = (np.abs(gabs) + np.abs(ref)) * 2.0 * 2.0 ** -8 if gabs is not None else 2.0 ** -6 * np.abs(ref)
    elt = err - (elt_atol + scale)
    _log("grad", dict(max=float(err.max()), rel_l2=r, elt_margin=float((err / (elt_atol + scale)).max()),
                      gate_a_max_frac=float(err.max() / atol_max) if gate_a else None,
                      q7_margin=float((err / (1e-3 + 2.0 ** -6 * np.abs(ref))).max())))
    assert elt.max() <= 0, f"elementwise gate exceeded by {elt.max():.3e}"
    if gate_a:
        assert err.max() <= atol_max, f"max-abs {err.max():.3e} > {atol_max}"
    return dict(max=float(err.max()), rel_l2=r)
