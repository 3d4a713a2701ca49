"""Host packing utilities of the product (paper_2504_02658_b200.pack) against
the oracle and the reference's golden vectors (bit-exact, CPU)."""
import os

import numpy as np
import pytest

from paper_2504_02658_b200 import pack as hp

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


def test_pack32_matches_golden():
    g = np.load(GOLD)
    assert (hp.pack_groups(g["pack32_in"]) == g["pack32_out"]).all()
    assert (hp.unpack_groups(g["pack32_out"]) == g["pack32_in"]).all()
    with pytest.raises(Exception):
        hp.pack32(np.full(32, 8, np.uint8))


@pytest.mark.parametrize("name", ["pm0", "pm1", "pm2"])
def test_pack_matrix_matches_golden(name):
    g = np.load(GOLD)
    codes, sc, ze = g[name + "_codes"], g[name + "_scales"], g[name + "_zeros"]
    for tiled in (0, 1):
        for split in (0, 1):
            key = f"{name}_t{tiled}s{split}"
            P = hp.pack_matrix(codes, sc, ze, tiled=bool(tiled), split=bool(split))
            if split:
                assert (P.plane_a == g[key + "_pa"]).all() and (P.plane_b == g[key + "_pb"]).all()
            else:
                assert (P.words == g[key + "_words"]).all()
            assert (P.scales == g[key + "_sh"]).all() and (P.zeros == g[key + "_zh"]).all()
            assert (hp.unpack_codes(P) == codes).all()
    Ps = hp.pack_matrix(codes, sc, None)
    assert (Ps.words == g[name + "_sym_words"]).all() and (Ps.scales == g[name + "_sym_sh"]).all()


def test_float_to_half_matches_golden():
    g = np.load(GOLD)
    got = hp.float_to_half_bits(g["f2h_in"])
    want = g["f2h_out"]
    nan = np.isnan(g["f2h_in"])
    assert (got[~nan] == want[~nan]).all()
