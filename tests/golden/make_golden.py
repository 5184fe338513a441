"""Writes tests/golden/*.json from closed forms evaluated with Python's math module only.

No value here comes from the CUDA path or from the oracle: these are the textbook
softmax cross-entropy formulas (PAPER.md line 273 / line 235: the fused LCE must
reproduce the "torch standard method", i.e. standard softmax CE) evaluated by hand
on a 2-token, 3-word example, plus ln V for each BASELINE.json vocabulary size
(the W = 0 closed form: every logit is 0, so lse = ln V and loss = ln V).
Run:  python tests/golden/make_golden.py
"""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def example_2x3():
    # X = [[1], [2]]  (N=2, H=1);  W = [[1], [0], [-1]]  (V=3);  targets t = [0, 2]
    # Z row 0 = [1, 0, -1];  Z row 1 = [2, 0, -2]
    S0 = math.e + 1.0 + math.exp(-1.0)
    S1 = math.exp(2.0) + 1.0 + math.exp(-2.0)
    lse0, lse1 = math.log(S0), math.log(S1)
    l0 = lse0 - 1.0          # target logit Z[0,0] = 1
    l1 = lse1 + 2.0          # target logit Z[1,2] = -2
    p0 = [math.e / S0, 1.0 / S0, math.exp(-1.0) / S0]
    p1 = [math.exp(2.0) / S1, 1.0 / S1, math.exp(-2.0) / S1]
    out = {"X": [[1.0], [2.0]], "W": [[1.0], [0.0], [-1.0]], "t": [0, 2], "lse": [lse0, lse1],
           "loss_rows": [l0, l1], "cases": {}}
    for red, c in (("sum", 1.0), ("mean", 0.5)):
        g0 = [c * (p0[0] - 1.0), c * p0[1], c * p0[2]]
        g1 = [c * p1[0], c * p1[1], c * (p1[2] - 1.0)]
        # dX_i = sum_v G_iv W_v ;  W = [1, 0, -1]
        dX = [[g0[0] - g0[2]], [g1[0] - g1[2]]]
        # dW_v = sum_i G_iv X_i ;  X = [1, 2]
        dW = [[g0[v] * 1.0 + g1[v] * 2.0] for v in range(3)]
        loss = (l0 + l1) * (1.0 if red == "sum" else 0.5)
        out["cases"][red] = {"loss": loss, "dX": dX, "dW": dW}
    out["cite"] = "closed form of standard softmax CE (PAPER.md l.273, l.235); derivation in make_golden.py"
    return out


def main():
    with open(os.path.join(HERE, "closed_form_2x3.json"), "w") as f:
        json.dump(example_2x3(), f, indent=1)
    lnv = {str(V): math.log(V) for V in (4096, 128256, 152064, 32768, 16032, 1)}
    with open(os.path.join(HERE, "w_zero_lnV.json"), "w") as f:
        json.dump({"cite": "W=0 => all logits 0 => loss = ln V (SURVEY §8(c) p2)", "lnV": lnv}, f, indent=1)


if __name__ == "__main__":
    main()
