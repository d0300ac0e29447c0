"""Write a 128-byte rsa_instance (the golden regression stream's parameters,
tests/golden/regression.json; p1 <= floor(sqrt q) as for every derived stream)
to tools/variants/inst_stream0.bin for sched_search.cu.  Host-only."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1811_11629_b200 import rsacore, skipgen
g = json.load(open(os.path.join(ROOT, "tests", "golden", "regression.json")))["params"]
p = rsacore.make_params(g["p1"], g["p2"], g["e"], skipgen.SkipParams.create(g["a"]))
rec = rsacore._instance_record(p)
open(os.path.join(ROOT, "tools", "variants", "inst_stream0.bin"), "wb").write(rec.tobytes())
print("wrote", rec.nbytes, "bytes; p1", p.p1, "p2", p.p2)
