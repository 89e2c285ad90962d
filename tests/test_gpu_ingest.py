"""GPU ingest path: files -> pinned batch -> H2D copies
overlapped with the fused pipeline (mtb_align_fused_ex + stream-ordered
ready flags).  Bit-exact against the oracle and against the in-memory path."""

import numpy as np
import pytest

import mtb_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mtb(cuda):
    import paper_2007_06483_b200 as m
    from paper_2007_06483_b200 import _lib

    _lib.load()
    return m


def _write_stack(m, tmp_path, w, h, count, seed, fmt="ppm"):
    rng = np.random.default_rng(seed)
    base = np.dstack([orc.synthetic_gray(rng, w, h) for _ in range(3)])
    imgs, _ = orc.generate_stack(base, count, seed=seed, max_shift=12)
    paths = []
    for i, im in enumerate(imgs):
        p = tmp_path / f"img{i}.{fmt if i % 2 == 0 else 'png'}"
        m.encode_image(im, p)
        paths.append(p)
    return imgs, paths


@pytest.mark.parametrize("w,h", [(512, 384), (1008, 700)])
def test_align_files_matches_oracle_and_align_stack(mtb, cuda, tmp_path, w, h):
    imgs, paths = _write_stack(mtb, tmp_path, w, h, 5, seed=w)
    aligned, rec = mtb.align_files(paths, workers=4)
    ref_aligned, ref_rec = mtb.align_stack(imgs)
    assert [r.offset for r in rec.pairwise] == [r.offset for r in ref_rec.pairwise]
    assert rec.cumulative == ref_rec.cumulative
    for a, b in zip(aligned, ref_aligned):
        np.testing.assert_array_equal(a, b)
    pre = [orc.preprocess(im, 6, 4) for im in imgs]
    for i, res in enumerate(rec.pairwise):
        want = orc.find_offset(pre[i]["mtb"], pre[i + 1]["mtb"])
        assert tuple(res.offset) == tuple(want["offset"])
        for tr, wt in zip(res.traces, want["traces"]):
            assert [e for _, e in tr.candidates] == [e for _, e in wt["candidates"]]
    assert set(rec.timings) == {"decode", "align", "shift"}


def test_align_files_pivot(mtb, cuda, tmp_path):
    imgs, paths = _write_stack(mtb, tmp_path, 640, 480, 5, seed=3)
    aligned, rec = mtb.align_files(paths, mode="pivot")
    ref_aligned, ref_rec = mtb.align(imgs, mode="pivot")
    assert rec.cumulative == ref_rec.cumulative
    for a, b in zip(aligned, ref_aligned):
        np.testing.assert_array_equal(a, b)


def test_streamed_fused_equals_resident(mtb, cuda):
    """align_fused_host (copies racing the pipeline) == align_fused on a resident batch."""
    torch = cuda
    imgs = []
    rng = np.random.default_rng(9)
    base = np.dstack([orc.synthetic_gray(rng, 1024, 768) for _ in range(3)])
    for i in range(4):
        a, _ = orc.generate_stack(base, 2, seed=20 + i, max_shift=30)
        imgs += a
    host = torch.from_numpy(np.stack(imgs)).pin_memory()
    eng = mtb.MtbEngine(1024, 768, 6, 4)
    pairs = [(2 * i, 2 * i + 1) for i in range(4)]
    for _ in range(3):   # repeated calls reuse the ready flags and copy stream
        dev, pyr_s, acc_s, errs_s = eng.align_fused_host(host, pairs)
        torch.cuda.synchronize()
        assert torch.equal(dev.cpu(), host)
        pyr_r, acc_r, errs_r = eng.align_fused(host.cuda(), pairs)
        torch.cuda.synchronize()
        assert torch.equal(acc_s, acc_r) and torch.equal(errs_s, errs_r)
        assert torch.equal(pyr_s.medians, pyr_r.medians)
        for i in range(len(imgs)):
            for k in range(eng.n):
                assert torch.equal(eng.bitmap_words(pyr_s.mtb, i, k), eng.bitmap_words(pyr_r.mtb, i, k))
                assert torch.equal(eng.bitmap_words(pyr_s.excl, i, k), eng.bitmap_words(pyr_r.excl, i, k))
