"""NEXT-4 pieces that do not need the (absent) Gset instance files: hex codec pinned to SPEC's
worked examples and to the lengths of the PAPER.md Appendix bitstrings, Gset round trip."""
import os

import numpy as np
import pytest

import synth
from paper_2311_09275_b200 import gset

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hex_examples_and_round_trip():
    assert list(gset.decode_hex("F", 4)) == [1, 1, 1, 1]
    assert list(gset.decode_hex("A", 4)) == [1, 0, 1, 0]        # S:204 (MSB first)
    assert gset.encode_hex([1, 1, 1, 1]) == "F"
    rng = np.random.default_rng(0)
    for n in list(range(1, 65)) + [10000]:
        b = rng.integers(0, 2, n).astype(np.uint8)
        assert np.array_equal(gset.decode_hex(gset.encode_hex(b), n), b)
    with pytest.raises(ValueError):
        gset.decode_hex("G1", 8)
    with pytest.raises(ValueError):
        gset.decode_hex("FF", 9)


def _hexfile(name):
    return "".join(l.strip() for l in open(os.path.join(GOLD, name)) if not l.startswith("#"))


def test_appendix_bitstrings_lengths():
    g72 = _hexfile("appendix_g72.hex")
    bits = gset.decode_hex(g72, 10000)                  # Appendix II: variables 1..10000
    assert bits.size == 10000
    assert gset.encode_hex(bits) == g72.upper()          # round trip of the paper's string
    g77 = _hexfile("appendix_g77.hex")
    with pytest.raises(ValueError):                      # truncated in PAPER.md
        gset.decode_hex(g77, 14000)


def test_gset_round_trip_and_host_cut():
    Jr, Jd = synth.torus_pm1(6, 4, 3)
    u, v, w = synth.torus_edges(6, 4, Jr, Jd)
    n2, u2, v2, w2 = gset.parse_gset(gset.write_gset(24, u, v, w))
    assert n2 == 24 and np.array_equal(u2, u) and np.array_equal(v2, v) and np.array_equal(w2, w)
    s = np.ones(24, np.int8)
    assert gset.cut_of(u, v, w, s) == 0
    s[0] = -1
    nb = (u == 0) | (v == 0)
    assert gset.cut_of(u, v, w, s) == int(w[nb].sum())


def test_parse_gset_rejects_malformed_files():
    """S:43-60 / S:29-35: truncated files, trailing tokens, self-loops and duplicate edges are
    errors naming the line (line 1 = header)."""
    import pytest
    from paper_2311_09275_b200.gset import parse_gset
    good = "3 2\n1 2 1\n2 3 -1\n"
    n, u, v, w = parse_gset(good)
    assert n == 3 and list(u) == [0, 1] and list(v) == [1, 2] and list(w) == [1, -1]
    with pytest.raises(ValueError, match="truncated"):
        parse_gset("3 2\n1 2 1\n2 3\n")
    with pytest.raises(ValueError, match="trailing"):
        parse_gset("3 2\n1 2 1\n2 3 -1\n7\n")
    with pytest.raises(ValueError, match="self-loop on line 3"):
        parse_gset("3 2\n1 2 1\n3 3 1\n")
    with pytest.raises(ValueError, match="duplicate edge on line 3"):
        parse_gset("3 2\n1 2 1\n2 1 1\n")
    with pytest.raises(ValueError, match="out of range on line 2"):
        parse_gset("3 1\n1 4 1\n")
