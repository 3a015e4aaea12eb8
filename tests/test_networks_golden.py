"""The comparator networks the oblivious kernels run are the verified ones (CPU).

tests/golden/networks.json holds, for every network the generated CUDA
programs execute (each stage after dead-code elimination, plus the column
sorts; paper_2507_19926_b200.netexport), the SHA-256 of its text in the
reference's network-file format (networks.py:603-641) and the result of the
reference's own zero-one verifier on it (networks.py:488-567), produced by
tools/verify_networks.py.  Regenerating must give exactly those networks, so
a code-generator change that alters any network fails here until it is
re-verified.
"""
import json
import os

import pytest

from paper_2507_19926_b200 import netexport

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "networks.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_every_network_verified_by_the_reference():
    doc = _golden()
    assert doc["all_ok"]
    assert all(r["ok"] for r in doc["networks"].values())
    modes = {r["mode"] for r in doc["networks"].values()}
    assert modes <= {"exhaustive", "random"}
    # everything up to 24 wires is proven exhaustively
    for name, r in doc["networks"].items():
        if r["wires"] <= 24:
            assert r["mode"] == "exhaustive", name


def test_generated_networks_match_the_verified_digests():
    doc = _golden()["networks"]
    got = netexport.export()
    assert {e["sha256"] for e in got.values()} == {r["sha256"] for r in doc.values()}
    for name, e in got.items():
        assert name in doc and doc[name]["sha256"] == e["sha256"], name


def test_network_text_is_reference_format():
    got = netexport.export()
    for e in list(got.values())[:20]:
        lines = [ln for ln in e["text"].splitlines() if ln and not ln.startswith("#")]
        assert lines[0].split()[0] == "WIRES"
        n = int(lines[0].split()[1])
        for ln in lines[1:]:
            op, i, j = ln.split()
            assert op in ("CE", "MIN", "MAX") and 0 <= int(i) < int(j) < n


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="the reference (build container only)")
def test_reference_reverifies_a_sample(tmp_path):
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from tilemedian import networks as refnet
    got = sorted(netexport.export().items(), key=lambda kv: kv[1]["wires"])[:12]
    for name, e in got:
        p = tmp_path / f"{name}.net"
        p.write_text(e["text"])
        net = refnet.load_network_file(p)
        c = e["claim"]
        claim = (refnet.Claim.sorted() if c["kind"] == "sorted"
                 else refnet.Claim.of_ranks({w: w for w in c["ranks"]}, c["runs"]))
        assert refnet.verify_zero_one(net, claim).ok, name
