"""NEXT-2 scene recipe (host logic): the twisting-rods generator matches Table 1's size (P:679,
355K tets / 70.4K nodes) and its scripted Dirichlet ends (torsion from both ends at 5/12
rev/s) are rigid rotations about the bundle axis in opposite directions."""
import numpy as np

import scenes


def test_twisting_rods_size_and_scripted_ends():
    sc = scenes.make_twisting_rods()
    assert len(sc["tets"]) == 355968 and len(sc["x0"]) == 70304  # paper: 355K / 70.4K
    fixed = sc["node_fixed"].astype(bool)
    assert np.array_equal(fixed, sc["twist_end"] > 0)
    h = sc["params"]["h"]
    w = sc["twist_omega"]
    assert abs(w * h - 2 * np.pi * 5 / 12 / 30) < 1e-15  # 5 degrees per frame
    x0 = sc["rest_x"]
    for k in (1, 7, 30):
        xt = scenes.twist_targets(sc, k * h)
        assert np.array_equal(xt[~fixed], x0[~fixed])
        for side, sign in ((1, 1.0), (2, -1.0)):
            m = sc["twist_end"] == side
            a0 = np.arctan2(x0[m, 1], x0[m, 0])
            a1 = np.arctan2(xt[m, 1], xt[m, 0])
            dang = np.angle(np.exp(1j * (a1 - a0)))
            assert np.allclose(dang, sign * w * k * h, atol=1e-12)
            np.testing.assert_allclose(np.hypot(xt[m, 0], xt[m, 1]), np.hypot(x0[m, 0], x0[m, 1]), rtol=1e-14)
            np.testing.assert_array_equal(xt[m, 2], x0[m, 2])
