"""Verification report on the GPU against the reference's
definitions (metrics.cpp, tools/mssz.cpp:69-104) recomputed from the oracle's
directions/labels, and against the reference's own known answers
(test_metrics.cpp).  Counts are exact; psnr within 1e-12 relative (the
reference's own test tolerance, test_metrics.cpp:40)."""
import math

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.fixture(scope="module")
def P(mssz):
    if mssz.library().mssz_cu_device_count() == 0:
        pytest.fail("no CUDA device visible to the GPU test suite")
    return mssz


def expected(oracle_lib, dims, f, g, xi, edit_count, archive_bytes):
    n = f.size
    fa, fd = oracle_lib.compute_directions(dims, f)
    ga, gd = oracle_lib.compute_directions(dims, g)
    fM, fm = oracle_lib.compute_labels(dims, fa, fd)
    gM, gm = oracle_lib.compute_labels(dims, ga, gd)
    mism = int(np.count_nonzero((fM != gM) | (fm != gm)))
    v = np.arange(n, dtype=np.uint64)
    c0 = (ga == v) & (fa != v)
    c1 = ~c0 & (gd == v) & (fd != v)
    c2 = ~c0 & ~c1 & (fa == v) & (ga != v)
    c3 = ~c0 & ~c1 & ~c2 & (fd == v) & (gd != v)
    d = f.astype(np.float64) - g.astype(np.float64)
    sq = math.fsum((d * d).tolist())
    lo, hi = float(f.astype(np.float64).min()), float(f.astype(np.float64).max())
    rmse = math.sqrt(sq / n)
    psnr = math.inf if rmse == 0 else 20.0 * math.log10((hi - lo) / rmse)
    rep = dict(mismatches=mism, mss_distortion=mism / n, psnr=psnr, edit_ratio=edit_count / n,
               bound_violations=int(np.count_nonzero(np.abs(d) > xi)),
               fp_max=int(c0.sum()), fp_min=int(c1.sum()), fn_max=int(c2.sum()), fn_min=int(c3.sum()))
    if archive_bytes:
        rep["ocr"] = n * f.itemsize / archive_bytes
        rep["obr"] = 8.0 * archive_bytes / n
    return rep


def check(rep, want):
    for k, v in want.items():
        got = getattr(rep, k)
        if k == "psnr" and math.isfinite(v):
            assert got == pytest.approx(v, rel=1e-12), k
        elif isinstance(v, float):
            assert got == v or got == pytest.approx(v, rel=1e-15), k
        else:
            assert got == v, k


@pytest.mark.parametrize("kind,dims,rel,dt", [
    ("gaussian-mixture", [128, 96], 1e-2, np.float32),
    ("random-smooth", [40, 36, 30], 1e-3, np.float32),
    ("trig", [33, 29, 17], 1e-2, np.float64),
])
def test_report_matches_definitions(P, oracle_lib, kind, dims, rel, dt):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate(kind, dims, 3, dt)
    xi = I.resolve_rel(f, rel)
    fh = I.compress_base(dims, f, xi)
    edits = P.derive_edits(topo, f, fh, xi, P.DeriveOptions(subloop_cap=100000))
    g = P.apply_edits(topo, fh, edits)
    # the corrected field: preserved segmentation, every bound kept
    rep = P.build_report(topo, f, g, xi, edits.size(), 12345)
    check(rep, expected(oracle_lib, dims, f, g, xi, edits.size(), 12345))
    assert rep.passed() and rep.mismatches == 0 and rep.fp_max + rep.fp_min + rep.fn_max + rep.fn_min == 0
    # the uncorrected decompressed field, and one with bound violations
    for cand in (fh, fh + np.asarray(2.5 * xi, dt) * (np.arange(fh.size) % 7 == 0)):
        cand = cand.astype(dt)
        rep = P.build_report(topo, f, cand, xi)
        check(rep, expected(oracle_lib, dims, f, cand, xi, 0, 0))


def test_report_reference_kats(P):
    # psnr closed forms (test_metrics.cpp:32-41)
    topo = P.build_topology([4, 4])
    f = np.array([(i % 2) * 1.0 for i in range(16)])
    assert math.isinf(P.build_report(topo, f, f, 0.5).psnr)
    assert P.build_report(topo, f, f + 0.1, 0.5).psnr == pytest.approx(20.0, rel=1e-12)
    # bound violation counting (test_metrics.cpp:85-90)
    topo = P.build_topology([2, 2])
    f = np.zeros(4)
    g = np.array([0.05, -0.05, 0.2, 0.0])
    assert P.build_report(topo, f, g, 0.1).bound_violations == 1
    assert P.build_report(topo, f, g, 0.01).bound_violations == 3
    # edit_ratio / ocr / obr (test_metrics.cpp:62-70)
    topo = P.build_topology([10, 10])
    f = np.arange(100, dtype=np.float64)
    r = P.build_report(topo, f, f, 1.0, 5, 800)
    assert r.edit_ratio == pytest.approx(0.05) and r.ocr == pytest.approx(1.0) and r.obr == pytest.approx(64.0)
    with pytest.raises(P.Error) as e:
        P.build_report(topo, f, f, 0.0)
    assert e.value.kind() == P.ErrKind.usage


def test_report_device_matches_host(P):
    import torch
    from paper_2406_09423_b200 import inputs as I
    dims = [64, 48, 40]
    topo = P.build_topology(dims)
    f = I.generate("multi-scale", dims, 2)
    xi = I.resolve_rel(f, 1e-3)
    fh = I.compress_base(dims, f, xi)
    host = P.build_report(topo, f, fh, xi)
    df, dg = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
    dev = P.build_report_device(topo, df.data_ptr(), dg.data_ptr(), xi, np.float32,
                                stream=torch.cuda.current_stream().cuda_stream)
    for k in ("mismatches", "bound_violations", "fp_max", "fp_min", "fn_max", "fn_min", "sum_sq", "psnr"):
        assert getattr(dev, k) == getattr(host, k), k


@pytest.mark.parametrize("dims,dt", [([177, 95, 48], np.float32), ([96, 64], np.float64),
                                     ([128, 32, 16], np.float32)])
def test_segmentation_matches_reference(P, golden, oracle_lib, dims, dt, tmp_path):
    from paper_2406_09423_b200 import inputs as I
    topo = P.build_topology(dims)
    f = I.generate("random-smooth", dims, 4, dt)
    lab = P.segmentation(topo, f)
    a, b = oracle_lib.compute_directions(dims, f)
    M, m = oracle_lib.compute_labels(dims, a, b)
    assert np.array_equal(lab.max_label, M) and np.array_equal(lab.min_label, m)
    out = tmp_path / "labels.bin"
    P.export_labels(lab, str(out))
    raw = np.frombuffer(out.read_bytes(), "<u8")
    assert np.array_equal(raw[:f.size], M) and np.array_equal(raw[f.size:], m)
    # the golden direction/label fields of the reference's own tests
    meta, arr = golden
    for case in meta["directions"]:
        p = f"dir/{case['name']}/"
        t = P.build_topology(case["dims"])
        lab = P.segmentation(t, arr[p + "values"])
        assert np.array_equal(lab.max_label, arr[p + "max_label"]), case["name"]
        assert np.array_equal(lab.min_label, arr[p + "min_label"]), case["name"]
