"""Golden reference_dot results (value, flexp_e, plain, or the exception) BY
RUNNING THE REFERENCE, for the device exact dot (paper_2105_00115_b200.exact).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_exact_golden.py

Inputs: every stored golden input (golden_inputs.npz) plus the edge vectors of
the reference's TestReferenceDot (test_kernel.py:72-122) and a few more
(signed zeros, subnormals, the Fraction-path triggers, overflow, non-finite).
Small special vectors are stored inline in the JSON.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from qdot.kernel import reference_dot  # noqa: E402


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64)]


def special():
    out = []
    rng = np.random.default_rng(9)
    out.append(("toy", [2.0**27, 2.0**8, 2.0**-3, 2.0**20], [2.0**23, 2.0**-14, 2.0**7, 2.0**-3]))
    out.append(("zeros", [0.0] * 5, [0.0] * 5))
    out.append(("neg_zero_products", [-0.0, 0.0, -0.0], [1.0, -2.0, 3.0]))
    out.append(("single_neg_zero", [-0.0], [5.0]))
    out.append(("cancellation", [1e16, 1.0, -1e16, 2.0**-30], [1.0] * 4))
    out.append(("plain_left_to_right", [1e16, 1.0, -1e16], [1.0] * 3))
    out.append(("huge_fallback", [1.7e308, 1.7e308, -1.7e308], [0.5, -0.5, 0.5]))
    out.append(("near_underflow", list(np.ldexp(rng.uniform(0.5, 1, 40), rng.integers(-530, -480, 40))),
                list(np.ldexp(rng.uniform(0.5, 1, 40), rng.integers(-530, -480, 40)))))
    out.append(("overflow", [1e308, 1e308], [1e308, 1e308]))
    out.append(("nonfinite", [1.0, float("inf")], [1.0, 1.0]))
    out.append(("nan", [1.0, float("nan")], [1.0, 1.0]))
    out.append(("subnormal_products", [5e-324, 2.0**-1070, -3e-320], [2.0**1000, 0.75, 2.0**600]))
    out.append(("subnormal_result", [2.0**-600, -2.0**-600], [2.0**-470, 2.0**-471]))
    out.append(("max_finite", [1.7976931348623157e308, -1.7976931348623157e308], [1.0, 0.5]))
    out.append(("tie_even", [1.0, 2.0**-53], [1.0, 1.0]))
    out.append(("tie_odd", [1.0 + 2.0**-52, 2.0**-53], [1.0, 1.0]))
    for seed in range(8):
        r = np.random.default_rng(seed)
        out.append((f"ldexp_normal_{seed}", list(np.ldexp(r.normal(size=100), r.integers(-40, 40, 100))),
                    list(np.ldexp(r.normal(size=100), r.integers(-40, 40, 100)))))
    r = np.random.default_rng(77)
    out.append(("wide_exponents", list(np.ldexp(r.normal(size=3000), r.integers(-1000, 1000, 3000))),
                list(np.ldexp(r.normal(size=3000), r.integers(-60, 10, 3000)))))
    return out


def record(name, x, y, stored_key=None):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    case = {"name": name}
    if stored_key:
        case["input"] = stored_key
    else:
        case["x"], case["y"] = hx(x), hx(y)
    try:
        r = reference_dot(x, y)
        case.update(raises=None, value=float(r.value).hex(), flexp_e=r.flexp_e, plain=float(r.plain).hex())
    except Exception as exc:  # noqa: BLE001
        case["raises"] = type(exc).__name__
    return case


def main():
    cases = [record(n, x, y) for n, x, y in special()]
    z = np.load(os.path.join(HERE, "golden_inputs.npz"))
    keys = sorted({k[:-3] for k in z.files if k.endswith("__x")})
    for k in keys:
        cases.append(record("stored_" + k, z[k + "__x"], z[k + "__y"], stored_key=k))
    with open(os.path.join(HERE, "exact_golden.json"), "w") as f:
        json.dump({"reference": "qdot 0.1.0 kernel.reference_dot", "cases": cases}, f, indent=0)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
