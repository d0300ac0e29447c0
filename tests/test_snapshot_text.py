"""Snapshot / params text is the reference's format byte for byte
(tests/golden/snapshot.json, written by the reference's rsacore)."""

import json
import os

import pytest

from paper_1811_11629_b200 import rsacore

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "snapshot.json")))


@pytest.mark.parametrize("case", sorted(GOLD))
def test_reference_text_round_trips(case):
    snap_text, params_text = GOLD[case]["snapshot"], GOLD[case]["params"]
    p = rsacore.params_from_text(params_text)
    assert rsacore.params_to_text(p) == params_text
    p2, st = rsacore.restore(snap_text)
    assert p2 == p
    assert rsacore.snapshot(st, p2).to_text() == snap_text
    assert rsacore.StreamSnapshot.from_text(snap_text).to_text() == snap_text


def test_malformed_texts_rejected():
    snap_text = GOLD["stream0_after_1234"]["snapshot"]
    bad = [snap_text.replace("rsarand-snapshot-v1", "rsarand-snapshot-v0"),
           snap_text.replace("\ndraws=", "\ndraws=zz"),
           snap_text.replace("m1=", "m9="),
           snap_text + "extra=1\n",
           snap_text.replace("\np1=", "\np1=1"),
           ""]
    for text in bad:
        with pytest.raises(rsacore.MalformedSnapshot):
            rsacore.restore(text)


@pytest.mark.gpu
def test_snapshot_after_draws_matches_reference():
    from paper_1811_11629_b200 import paramfactory
    p = paramfactory.derive_stream_params(paramfactory.StreamKey(paramfactory.DEFAULT_MASTER_SEED, 0))
    st = rsacore.init(p)
    rsacore.take_raws(st, p, 1234)
    assert rsacore.snapshot(st, p).to_text() == GOLD["stream0_after_1234"]["snapshot"]
    pc = rsacore.make_params(p.p1, p.p2, 9, p.skip, skip_mode=rsacore.SKIP_CONST, skip_const=12345)
    sc = rsacore.init(pc)
    rsacore.take_raws(sc, pc, 7)
    assert rsacore.snapshot(sc, pc).to_text() == GOLD["const_after_7"]["snapshot"]
