"""BASELINE config 2 (isolated batched kernels) on the B200 against the CPU
oracle on the same seeded blocks."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_batched_qr_matches_oracle():
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.batched import batched_qr, config2_inputs
    Bs, Cs, _ = config2_inputs(n_qr=96, n_rrqr=0)
    Rs, Co, ms = batched_qr(Bs, Cs)
    for B, Cm, R, HtC in zip(Bs, Cs, Rs, Co):
        V, tau, Rr = O.house_qr(B)
        assert np.abs(R - Rr).max() <= 1e-12 * np.abs(Rr).max()
        ref = O.wy_apply(V, O.larft(V, tau), Cm, True)
        assert np.abs(HtC - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_batched_rrqr_ranks_and_oracle():
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.batched import batched_rrqr, config2_inputs
    _, _, Ms = config2_inputs(n_qr=0, n_rrqr=64)
    for eps, lo, hi in ((1e-2, 16, 20), (1e-4, 33, 37)):
        ranks, rdiag, ms = batched_rrqr(Ms, eps)
        assert lo <= ranks.min() and ranks.max() <= hi
        for i in range(0, 64, 7):
            res = O.rrqr_threshold(Ms[i], eps)
            # sigma_16 / sigma_32 sit exactly on the tolerances:
            # a rank may differ by one only when the deciding norm is within
            # 1e-8 of the threshold
            d = np.abs(np.diag(res["R"][:, :res["rank"]]))
            if ranks[i] != res["rank"]:
                r = min(ranks[i], res["rank"])
                full = O.rrqr_threshold(Ms[i], 0.0)
                nd = np.abs(np.diag(full["R"]))
                assert abs(nd[r] / (eps * nd[0]) - 1.0) <= 1e-8
            k = min(ranks[i], res["rank"])
            assert np.allclose(rdiag[i, :k], d[:k], rtol=1e-10, atol=0)
