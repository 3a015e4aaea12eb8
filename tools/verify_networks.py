"""Verify every network the oblivious kernels run with the REFERENCE's verifier.

    PYTHONPATH=/root/reference/pkg/src python tools/verify_networks.py [--out tests/golden/networks.json]

Build-container only (the reference is not on the GPU box).  For each network
exported by paper_2507_19926_b200.netexport (the generated programs' stages as
the kernels execute them, plus the column sorts): write it in the reference's
network-description format, load it back with the reference's
``load_network_file`` (networks.py:612-632) and check its claim with the
reference's ``verify_zero_one`` (networks.py:488-567) -- exhaustive over the
0/1 input family when that has at most 2^24 members, else 20,000 random
inputs (which can only refute).  Writes the results, keyed by each network's
SHA-256, to tests/golden/networks.json; tests/test_networks_golden.py pins the
generator to them.
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from tilemedian import networks as refnet  # noqa: E402  (the reference itself)

from paper_2507_19926_b200 import netexport  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "networks.json"))
    ap.add_argument("--trials", type=int, default=20000)
    ap.add_argument("--dump", default=None, help="also keep the .net files in this directory")
    a = ap.parse_args()
    nets = netexport.export()
    results = {}
    t0 = time.time()
    with tempfile.TemporaryDirectory() as tmp:
        d = a.dump or tmp
        os.makedirs(d, exist_ok=True)
        for name, e in sorted(nets.items()):
            path = os.path.join(d, name + ".net")
            with open(path, "w") as f:
                f.write(e["text"])
            net = refnet.load_network_file(path)
            c = e["claim"]
            if c["kind"] == "sorted":
                claim = refnet.Claim.sorted()
            else:
                claim = refnet.Claim.of_ranks({w: w for w in c["ranks"]}, c["runs"])
            r = refnet.verify_zero_one(net, claim, max_evaluations=1 << 24,
                                       random_trials=a.trials, seed=0)
            results[name] = {"sha256": e["sha256"], "wires": e["wires"], "ops": e["ops"],
                             "claim": c["kind"] + (" over runs " + "+".join(map(str, c["runs"]))
                                                   if c["runs"] else ""),
                             "live_outputs": len(c["ranks"]) if c["ranks"] else e["wires"],
                             "ok": bool(r.ok), "mode": r.mode, "inputs_checked": int(r.inputs_checked),
                             "used_by": sorted(e["used_by"])}
            print(f"{name:36s} {e['wires']:4d}w {e['ops']:5d} ops  {r.mode:10s} "
                  f"{r.inputs_checked:9d}  {'ok' if r.ok else 'FAIL ' + r.detail}", flush=True)
    doc = {"generator": "paper_2507_19926_b200.netexport.export()",
           "verifier": "reference tilemedian.networks.verify_zero_one (networks.py:488-567), "
                       "max_evaluations=2^24, random_trials=%d" % a.trials,
           "seconds": round(time.time() - t0, 1),
           "all_ok": all(r["ok"] for r in results.values()),
           "networks": results}
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print("all ok" if doc["all_ok"] else "FAILURES", len(results), "networks", file=sys.stderr)


if __name__ == "__main__":
    main()
