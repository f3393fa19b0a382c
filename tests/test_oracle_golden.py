"""Pin the CPU oracle (oracle/seqref.py) to the reference itself: the
reference CLI's selftest parity dumps and the reference's live collective
algorithms on seeded inputs (tests/golden/, made by oracle/make_golden.py)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import seqref


@pytest.mark.parametrize("p", [2, 4, 8])
def test_oracle_matches_reference_selftest_dump(p):
    cases = gc.load_selftest(p)
    assert len(cases) == 78, "reference selftest dump: 13 kinds x 2 dtypes x 3 counts"
    for case in cases:
        got = gc.selftest_oracle(case, p)
        for r in range(p):
            want = case["expected"][r]
            g = got[r]
            if g is None:  # rooted op, non-root rank: the dump records []
                assert len(want) == 0
                continue
            seqref.assert_matches(g, np.asarray(want, dtype=g.dtype),
                                  where=f"p{p}/{case['op']}/{case['dtype']}/{case['count']}/r{r}")


def test_oracle_matches_reference_live_algorithms():
    cases = gc.load_live()
    assert len(cases) >= 600
    checked = 0
    for c in cases:
        want = c["outputs"]
        got = gc.live_oracle(c)
        for r in range(c["p"]):
            w, g = want[r], got[r]
            if w is None:
                continue
            where = f"{c['kind']}/p{c['p']}/{c['dtype']}/{c['count']}/{c['policy']}/r{r}"
            if c["kind"] == "all_to_all":
                for j, (wb, gb) in enumerate(zip(w, g)):
                    seqref.assert_matches(gb, gc.dec(wb), where=f"{where}[{j}]")
                continue
            wa = gc.dec(w)
            if c["policy"] == "ring":
                # ring folds in a different order: tolerance rule (cases.py:232-236)
                seqref.assert_matches(g, wa, float_reduction=True, rtol=1e-5, where=where)
            else:
                seqref.assert_matches(g, wa, where=where)  # naive = ascending fold: exact
            checked += 1
    assert checked > 1500


def test_trunc16_matches_reference_codec_and_compressed_collectives():
    """seqref.trunc16 against the reference Trunc16Codec round trip (specials
    included: +-0, +-inf, nan, denormals) and every compressible kind run by
    the reference's live algorithms with CompressionConfig at p=3."""
    g = gc.load_trunc16()
    assert g, "tests/golden/trunc16.json missing (python oracle/make_golden.py trunc16)"
    x, want = gc.dec(g["roundtrip"]["input"]), gc.dec(g["roundtrip"]["output"])
    got = seqref.trunc16(x)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    checked = 0
    for c in g["cases"]:
        got = gc.trunc16_oracle(c)
        for r in range(c["p"]):
            w = c["outputs"][r]
            if w is None:
                continue
            where = f"trunc16/{c['kind']}/{c['count']}/r{r}"
            if c["kind"] == "all_to_all":
                for j, wb in enumerate(w):
                    assert np.array_equal(got[r][j].view(np.uint32), gc.dec(wb).view(np.uint32)), where
            else:
                assert np.array_equal(np.asarray(got[r]).view(np.uint32),
                                      gc.dec(w).view(np.uint32)), where
            checked += 1
    assert checked >= 60


def test_known_answers_spec_examples():
    # test_collectives.py:39-117 and frontend partner.py known answers
    assert seqref.all_reduce([np.array([r, 2 * r], np.float64) for r in range(4)],
                             "sum")[0].tolist() == [6.0, 12.0]
    ins = [np.arange(c, dtype=np.int64) + 10 * c for c in (1, 2, 3)]
    assert seqref.all_gatherv(ins, [1, 2, 3], [0, 1, 3])[0].tolist() == [10, 20, 21, 30, 31, 32]
    g = seqref.gatherv([np.array([1.0, 2.0], np.float32), np.zeros(0, np.float32),
                        np.array([3.0], np.float32)], 0, [2, 0, 1], [0, 2, 2])
    assert g[0].tolist() == [1.0, 2.0, 3.0]
    assert [o.tolist() for o in seqref.all_to_all_single(
        [np.array([10, 11]), np.array([20, 21])])] == [[10, 20], [11, 21]]
    out = seqref.all_to_allv([np.array([1, 2, 3]), np.array([4, 5, 6])], [[1, 2], [2, 1]],
                             [[0, 1], [0, 2]], [[0, 1], [0, 2]])
    assert [o.tolist() for o in out] == [[1, 4, 5], [2, 3, 6]]


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 1e3,
                        np.array([0.0, -0.0, np.inf, -np.inf, 1e-40, 3.4e38], np.float32)])
    ours = seqref.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)
    assert np.isnan(seqref.bf16_bits_to_f32(seqref.f32_to_bf16_bits(np.array([np.nan], np.float32))))


def test_bf16_fold_is_f32_accumulate_then_one_rounding():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    ins = [seqref.f32_to_bf16_bits(rng.standard_normal(4096).astype(np.float32)) for _ in range(8)]
    got = seqref.fold_bf16(ins, "sum")
    acc = torch.zeros(4096, dtype=torch.float32)
    for b in ins:
        acc = acc + torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).float()
    want = acc.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(got, want)


def test_integer_wrap_like_c():
    a = np.array([2 ** 62, -5, 127], np.int64)
    b = np.array([4, -2 ** 63, 1], np.int64)
    with np.errstate(over="ignore"):
        assert seqref.fold([a, b], "prod")[0] == 0  # 2^64 wraps
    u = [np.array([200], np.uint8), np.array([100], np.uint8)]
    assert seqref.fold(u, "sum")[0] == 44 and seqref.fold(u, "prod")[0] == (200 * 100) % 256


def test_assert_matches_tolerance_rule():
    want = np.array([1000.0, 1.0], np.float32)
    got = want + np.array([0.009, 0.009], np.float32)  # atol = 1e-5 * 1000
    seqref.assert_matches(got, want, float_reduction=True, rtol=1e-5)
    with pytest.raises(AssertionError):
        seqref.assert_matches(got, want)  # bit-exact otherwise
