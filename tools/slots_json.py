"""Write profiles/slots.json: fmaheavy-datapath slots per draw of each fill /
fused kernel, counted from the SASS of the built library (tools/sass_slots.py
weights: IMAD.WIDE/HI 2, other IMAD 1, FP64 ops 1).  bench.py reports the
dominant kernel's achieved slot rate against the in-run probe peak."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
LIB = os.path.join(ROOT, "paper_1811_11629_b200", "librsarand_b200.so")


def count(fn: str, per_store: int = 0) -> float:
    """Heavy slots of the hot loop; divided by the draws per loop body when
    per_store > 0 (draws = per_store x the 128-bit streaming stores in the
    loop, so unrolled loops count right)."""
    txt = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True).stdout
    lines = [l for l in txt.splitlines() if re.search(r"/\*[0-9a-f]{4}\*/", l)]
    path = "/tmp/_slots.txt"
    with open(path, "w") as fh:
        fh.write("\n".join(lines))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_slots.py"), path, "--lightest"],
                         capture_output=True, text=True).stdout.splitlines()
    heavy = float(re.search(r"heavy slots ([0-9.]+)", out[0]).group(1))
    if per_store:
        stores = sum(int(l.split()[0]) for l in out[1:] if l.split()[1].startswith("STG.E.EF.128"))
        return heavy / (per_store * stores)
    return heavy


res = {}
for e in (3, 5, 9, 17, 65537):
    res[f"fill_e{e}"] = count(f"_ZN3rsa11k_fill_fastILj{e}ELi2ELb0ELi1EEEvPK12rsa_instancejmmPmS4_S4_S4_Pdmj",
                              per_store=2)
    res[f"fused_e{e}"] = None
for e in (3, 5, 9, 17):
    try:
        # the fused inner loop is unrolled by 2 (two draws per body)
        res[f"fused_e{e}"] = count(f"_ZN3rsa7k_fusedILj{e}EEEvPK12rsa_instancejmPmS4_S4_P14rsa_fused_statPj") / 2
    except Exception:
        pass
res["note"] = "slots per draw in the hot loop; 64 slots/clk/SM nominal"
with open(os.path.join(ROOT, "profiles", "slots.json"), "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res, indent=1))
