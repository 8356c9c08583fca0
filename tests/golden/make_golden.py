"""Extract the reference's own golden vectors into committed fixtures.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It parses, without executing anything from the reference:
  * proj/tests/test_rf3.cpp:29-45  kGolden (rf3_coefficients at 5 sigmas,
    frozen from a 50-digit evaluation)
  * proj/test_output.txt:9,11,14,16,17 the reference's captured acceptance
    numbers (criterion-1 impulse errors, criterion-3 DC gains, criterion-9
    anisotropy ratio, criterion-8 timings used only as the CPU baseline
    context)
and writes tests/golden/reference_golden.json. The GPU box never reads
/root/reference; tests read only the JSON.
"""
import json
import os
import re

REF = "/root/reference/proj"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def kgolden():
    src = open(os.path.join(REF, "tests/test_rf3.cpp")).read()
    block = src[src.index("constexpr Golden kGolden[] = {"):]
    block = block[: block.index("};")]
    rows = re.findall(r"\{([^{}]+)\}", block)
    keys = ["sigma", "a0", "a1", "a2", "a3", "alpha1", "alpha2", "alpha3", "beta"]
    out = []
    for r in rows:
        vals = [float(v) for v in r.replace("\n", " ").split(",") if v.strip()]
        assert len(vals) == 9, r
        out.append(dict(zip(keys, vals)))
    return {"source": "proj/tests/test_rf3.cpp:29-45", "rows": out}


def acceptance():
    txt = open(os.path.join(REF, "test_output.txt")).read()
    res = {"source": "proj/test_output.txt"}
    m = re.search(r"err1=([\d.e+-]+) err5=([\d.e+-]+) err10=([\d.e+-]+) err3=([\d.e+-]+)", txt)
    res["criterion1_impulse_l2"] = {"err1": float(m.group(1)), "err5": float(m.group(2)),
                                    "err10": float(m.group(3)), "err3": float(m.group(4)),
                                    "line": "test_output.txt:9"}
    m = re.search(r"worst rel err=([\d.e+-]+)", txt)
    res["criterion2_worst_rel"] = float(m.group(1))
    gains = re.findall(r"sigma=(\d+): g1=([\d.e+-]+) g3=([\d.e+-]+) \(want ([\d.e+-]+)\)", txt)
    res["criterion3_dc"] = [{"sigma": float(s), "g1": float(a), "g3": float(b), "want": float(w)}
                            for s, a, b, w in gains]
    m = re.search(r"ratio=([\d.e+-]+) want 3.5", txt)
    res["criterion9_ratio"] = float(m.group(1))
    m = re.search(r"t3=([\d.e+-]+)s t5=([\d.e+-]+)s t10=([\d.e+-]+)s", txt)
    res["criterion8_seconds_1024sq_1thread"] = {"t3": float(m.group(1)), "t5": float(m.group(2)),
                                                "t10": float(m.group(3))}
    m = re.search(r"worst dot-test=([\d.e+-]+).*B asymmetry=([\d.e+-]+).*min eigenvalue=([\d.e+-]+)",
                  txt)
    res["criterion6"] = {"worst_dot": float(m.group(1)), "asym": float(m.group(2)),
                         "min_eig": float(m.group(3))}
    return res


if __name__ == "__main__":
    data = {"kGolden": kgolden(), "acceptance": acceptance()}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", OUT)
