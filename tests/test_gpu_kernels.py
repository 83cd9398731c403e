"""GPU parity of the unit kernels against the fp64 CPU oracle
(oracle/gemm_oracle.c) on the same (rounded) inputs.

Tolerances (stated here): relative Frobenius error against the
fp64 oracle on the SAME rounded inputs <= 2e-5 for every unit; generator and
RNE conversions bit-exact.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-5


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _dev_fill(torch, poas, rows, cols, seed, dtype=None, ld=None):
    ld = ld or cols
    t = torch.empty(rows, ld, device="cuda", dtype=torch.float32)
    poas.fill_uniform(poas.DTYPE_F32, t.data_ptr(), ld, rows, cols, 0, 0, cols, seed)
    return t


def test_device_generator_bit_identical_to_oracle(torch_cuda, poas):
    import oracle

    torch = torch_cuda
    seed = poas.stream_seed(20261017, "A")
    assert seed == oracle.stream_seed(20261017, "A")
    for rows, cols, r0, c0, tot in [(37, 53, 0, 0, 53), (64, 64, 5, 7, 1000), (1, 4096, 3, 0, 4096)]:
        t = torch.empty(rows, cols, device="cuda")
        poas.fill_uniform(poas.DTYPE_F32, t.data_ptr(), cols, rows, cols, r0, c0, tot, seed)
        ref = oracle.fill_uniform(rows, cols, seed, r0, c0, tot)
        assert np.array_equal(t.cpu().numpy(), ref)
        host = np.empty((rows, cols), dtype=np.float32)
        poas.fill_uniform_host(host.ctypes.data, cols, rows, cols, r0, c0, tot, seed)
        assert np.array_equal(host, ref)
        for dt, mode in ((poas.DTYPE_BF16, 2), (poas.DTYPE_F16, 1)):
            td = torch.bfloat16 if dt == poas.DTYPE_BF16 else torch.float16
            h = torch.empty(rows, cols, device="cuda", dtype=td)
            poas.fill_uniform(dt, h.data_ptr(), cols, rows, cols, r0, c0, tot, seed)
            assert np.array_equal(h.float().cpu().numpy(), oracle.round_to(ref, mode))


def test_convert_rne_bit_identical(torch_cuda, poas):
    import oracle

    torch = torch_cuda
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((257, 129)) * 10.0 ** rng.integers(-6, 4, (257, 129))).astype(np.float32)
    src = torch.from_numpy(x).cuda()
    for dt, mode, td in ((poas.DTYPE_BF16, 2, torch.bfloat16), (poas.DTYPE_F16, 1, torch.float16)):
        out = torch.empty(257, 136, device="cuda", dtype=td)
        poas.convert_f32(dt, src.data_ptr(), 129, out.data_ptr(), 136, 257, 129)
        torch.cuda.synchronize()
        got = out[:, :129].float().cpu().numpy()
        assert np.array_equal(got, oracle.round_to(x, mode))


TC_SHAPES = [(128, 256, 64), (1000, 1000, 1000), (129, 300, 72), (64, 4096, 512), (4096, 64, 1024),
             (1, 1, 8), (7, 1000, 24), (255, 257, 136), (2048, 2048, 2048), (333, 1536, 4104)]


@pytest.mark.parametrize("variant", [None, "2cta512"])
@pytest.mark.parametrize("shape", TC_SHAPES)
@pytest.mark.parametrize("dtype,mode", [(2, 2), (1, 1)])
def test_tc_gemm_vs_oracle(torch_cuda, poas, monkeypatch, shape, dtype, mode, variant):
    """bf16 and fp16 operands, every shape through the size-chosen kernel and
    through the 256 x 512 pair tiles (tiny, ragged and long-K shapes)."""
    import oracle

    torch = torch_cuda
    if variant:
        monkeypatch.setenv("POAS_TC_KERNEL", variant)
    m, n, k = shape
    A = oracle.fill_uniform(m, k, 11)
    B = oracle.fill_uniform(k, n, 12)
    lda, ldb = (k + 7) // 8 * 8, (n + 7) // 8 * 8
    td = torch.bfloat16 if dtype == 2 else torch.float16
    a = torch.zeros(m, lda, device="cuda", dtype=td)
    b = torch.zeros(k, ldb, device="cuda", dtype=td)
    a[:, :k] = torch.from_numpy(A).cuda().to(td)
    b[:, :n] = torch.from_numpy(B).cuda().to(td)
    c = torch.full((m, n), float("nan"), device="cuda")
    poas.tc_gemm(dtype, m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), n)
    torch.cuda.synchronize()
    ref = oracle.gemm_rows_f64(A, B, mode)
    got = c.cpu().numpy()
    assert oracle.rel_frobenius(got, ref) <= TOL
    # against the UNROUNDED fp32 inputs: the operand
    # rounding dominates -- bf16 <= 8e-3, fp16 <= 2e-3; a statistical bound
    # (rounding errors average over K), so only from K >= 64 (at K = 8 one
    # 1x1 output can sit at 1.4e-2 for bf16)
    if k >= 64:
        exact = oracle.gemm_rows_f64(A, B, 0)
        assert oracle.rel_frobenius(got, exact) <= (8e-3 if dtype == 2 else 2e-3)


@pytest.mark.parametrize("ctas", [1, 2, 7, 146])
def test_tc_gemm_sm_budget_and_accumulate(torch_cuda, poas, ctas):
    import oracle

    torch = torch_cuda
    m, n, k = 700, 900, 264
    A, B = oracle.fill_uniform(m, k, 3), oracle.fill_uniform(k, n, 4)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(np.pad(B, ((0, 0), (0, 4)))).cuda().bfloat16()
    c0 = oracle.fill_uniform(m, n, 5)
    c = torch.from_numpy(c0).cuda()
    poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n + 4, c.data_ptr(), n, accumulate=True,
                 num_ctas=ctas)
    torch.cuda.synchronize()
    ref = oracle.gemm_rows_f64(A, B, 2) + c0.astype(np.float64)
    assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL


def test_tc_gemm_rejects_misaligned_pitch(torch_cuda, poas):
    from paper_2209_10245_b200 import PoasError

    torch = torch_cuda
    a = torch.zeros(16, 20, device="cuda", dtype=torch.bfloat16)
    c = torch.zeros(16, 20, device="cuda")
    with pytest.raises(PoasError) as e:  # 20 bf16 = 40 B row pitch: not a TMA 16 B multiple
        poas.tc_gemm(2, 16, 20, 20, a.data_ptr(), 20, a.data_ptr(), 20, c.data_ptr(), 20)
    assert e.value.errc == "cuda"


SIMT_SHAPES = [(128, 128, 16), (1000, 1000, 1000), (129, 300, 72), (77, 33, 5), (1, 5000, 777),
               (3, 4096, 1024), (8, 16384, 256), (16, 1030, 64), (17, 999, 33), (127, 513, 100),
               (2048, 2048, 2048)]


@pytest.mark.parametrize("shape", SIMT_SHAPES)
@pytest.mark.parametrize("ctas", [0, 2])
def test_simt_gemm_vs_oracle(torch_cuda, poas, shape, ctas):
    import oracle

    torch = torch_cuda
    m, n, k = shape
    A, B = oracle.fill_uniform(m, k, 21), oracle.fill_uniform(k, n, 22)
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.full((m, n), float("nan"), device="cuda")
    poas.simt_gemm(m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, num_ctas=ctas,
                   exclusive=ctas > 0)
    torch.cuda.synchronize()
    ref = oracle.gemm_rows_f64(A, B, 0)
    assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL


SIMT_VARIANTS = ["ffma2", "ffma2k32", "ffma2k16", "ffma2k16j", "ffma2x2", "ffma2w16", "ffma2x512", "256", "128"]


@pytest.mark.parametrize("variant", SIMT_VARIANTS)
@pytest.mark.parametrize("shape", [(1000, 1000, 1000), (129, 300, 72), (640, 1024, 512), (333, 777, 100)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_simt_variants_vs_oracle(torch_cuda, poas, monkeypatch, variant, shape, accumulate):
    """Every CUDA-core kernel variant (POAS_SIMT_TILE, read per launch) on
    square, ragged and strided shapes, overwrite and accumulate."""
    import oracle

    torch = torch_cuda
    monkeypatch.setenv("POAS_SIMT_TILE", variant)
    m, n, k = shape
    lda, ldb = k + (4 if m % 2 else 0), n + (8 if n % 2 else 0)
    A, B = oracle.fill_uniform(m, lda, 31), oracle.fill_uniform(k, ldb, 32)
    C0 = oracle.fill_uniform(m, n, 33)
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.from_numpy(C0).cuda() if accumulate else torch.full((m, n), float("nan"), device="cuda")
    poas.simt_gemm(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), n, accumulate=accumulate)
    torch.cuda.synchronize()
    ref = oracle.gemm_rows_f64(A[:, :k], B[:, :n], 0) + (C0 if accumulate else 0)
    assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL


def test_simt_accumulate_and_strided(torch_cuda, poas):
    import oracle

    torch = torch_cuda
    m, n, k = 300, 500, 96
    A, B, C0 = oracle.fill_uniform(m, k + 3, 1), oracle.fill_uniform(k, n + 5, 2), oracle.fill_uniform(m, n, 3)
    a, b, c = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.from_numpy(C0).cuda()
    poas.simt_gemm(m, n, k, a.data_ptr(), k + 3, b.data_ptr(), n + 5, c.data_ptr(), n, accumulate=True)
    torch.cuda.synchronize()
    ref = oracle.gemm_rows_f64(A[:, :k], B[:, :n], 0) + C0
    assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL


def test_full_size_tc_property(torch_cuda, poas):
    """BASELINE size (16384^3): size-independent check C.x == A.(B.x) for a
    random x, in fp64 on the device, on the rounded bf16 inputs."""
    torch = torch_cuda
    n = 16384
    sa, sb = poas.stream_seed(20261017, "A"), poas.stream_seed(20261017, "B")
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, sa)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, sb)
    c = torch.empty(n, n, device="cuda")
    poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n)
    torch.cuda.synchronize()
    x = torch.randn(n, 4, device="cuda", dtype=torch.float64)
    rhs = a.double() @ (b.double() @ x)
    rel = ((c.double() @ x - rhs).norm() / rhs.norm()).item()
    # fp32 accumulation over K = 16384 on the tensor pipe: the stated bound
    # grows with K; cuBLAS on the same inputs for scale
    tol = TOL * max(1.0, n / 16384)
    assert rel <= tol, rel
    ref = torch.mm(a, b, out_dtype=torch.float32)
    rel_cublas = ((ref.double() @ x - rhs).norm() / rhs.norm()).item()
    assert rel <= 1.5 * rel_cublas + 1e-6, (rel, rel_cublas)


@pytest.mark.parametrize("variant", ["1cta", "2cta", "2cta512", "2cta512x2", "2cta256x2"])
def test_tc_kernel_forward_k_order(torch_cuda, poas, monkeypatch, variant):
    """POAS_TC_KSERP=0: every tile sweeps K forwards (the default alternates
    the direction per wave of tiles); both orders agree with the oracle and
    with each other to fp32 accumulation-order rounding."""
    import oracle

    torch = torch_cuda
    monkeypatch.setenv("POAS_TC_KERNEL", variant)
    m, n, k = 1500, 1304, 1000
    A, B = oracle.fill_uniform(m, k, 41), oracle.fill_uniform(k, n, 42)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    out = []
    for ks in ("0", "1"):
        monkeypatch.setenv("POAS_TC_KSERP", ks)
        c = torch.full((m, n), float("nan"), device="cuda")
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, num_ctas=8)
        torch.cuda.synchronize()
        assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL, ks
        out.append(c)
    assert ((out[0] - out[1]).abs().max() / out[0].abs().max()).item() < 1e-5


# (variant, epilogue): the single-SM kernels have one epilogue
_TC_VARIANTS = [("1cta", "tma"), ("1cta128", "tma"), ("1cta64", "tma"), ("2cta", "tma"), ("2cta", "direct"),
                ("2cta", "tma-epi8"), ("2cta", "direct-epi8"), ("2cta", "tma-epi4"),
                ("2cta512", "tma"), ("2cta512", "direct"), ("2cta512x2", "tma"),
                ("2cta512x2", "direct"), ("2cta256x2", "tma"), ("2cta256x2", "direct")]


@pytest.mark.parametrize("sched", ["dynamic", "static", "wave"])
@pytest.mark.parametrize("variant,epilogue", _TC_VARIANTS)
@pytest.mark.parametrize("shape", [(300, 520, 200), (256, 256, 64), (1000, 1000, 1000), (2049, 777, 136)])
def test_tc_kernel_variants(torch_cuda, poas, monkeypatch, variant, shape, sched, epilogue):
    """The tensor kernels (single-SM 128x256 / 128x128 / 128x64, CTA-pair
    256x256 with 4 or 8 epilogue warps and 256x512) under
    every tile scheduler and both pair-kernel epilogues (TMA store; direct
    register stores) agree with the oracle, including partial pair tiles,
    odd SM budgets and a C pitch TMA cannot map (n = 777)."""
    import oracle

    torch = torch_cuda
    monkeypatch.setenv("POAS_TC_KERNEL", variant)
    monkeypatch.setenv("POAS_TC_SCHED", sched)
    epilogue, _, epi = epilogue.partition("-epi")  # the 256x256 kernel's epilogue warps
    if epilogue != "tma":
        monkeypatch.setenv("POAS_TC_EPILOGUE", epilogue)
    if epi:
        monkeypatch.setenv("POAS_TC_EPI", epi)
    m, n, k = shape
    A, B = oracle.fill_uniform(m, k, 31), oracle.fill_uniform(k, n, 32)
    ldb = (n + 7) // 8 * 8
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.zeros(k, ldb, device="cuda", dtype=torch.bfloat16)
    b[:, :n] = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    for ctas in (0, 3, 10):
        c = torch.full((m, n), float("nan"), device="cuda")
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), ldb, c.data_ptr(), n, num_ctas=ctas)
        torch.cuda.synchronize()
        assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL, (variant, ctas)


@pytest.mark.parametrize("variant", [None, "2cta512", "2cta512x2"])
@pytest.mark.parametrize("accumulate", [False, True])
def test_tc_epilogue_pitch_and_alignment(torch_cuda, poas, monkeypatch, accumulate, variant):
    """C inside a wider buffer: a padded pitch (TMA-store epilogue, tails
    clipped: the padding is never written) and a 4-byte-offset base (no
    tensor map: direct stores); both plain and accumulating (TMA f32 add
    reduction)."""
    import oracle

    torch = torch_cuda
    if variant:
        monkeypatch.setenv("POAS_TC_KERNEL", variant)
    m, n, k = 700, 600, 320
    A, B = oracle.fill_uniform(m, k, 41), oracle.fill_uniform(k, n, 42)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    for pad, off in ((8, 0), (5, 1)):
        big = torch.full((m, n + pad), float("nan") if not accumulate else 0.0, device="cuda")
        if accumulate:
            big[:, off:off + n] = 1.0
        c = big[:, off:off + n]
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n + pad,
                     accumulate=accumulate)
        torch.cuda.synchronize()
        got = c.cpu().numpy() - (1.0 if accumulate else 0.0)
        assert oracle.rel_frobenius(got, ref) <= TOL, (pad, off)
        rest = torch.cat([big[:, :off], big[:, off + n:]], dim=1).cpu().numpy()
        if accumulate:
            assert (rest == 0.0).all()
        else:
            assert np.isnan(rest).all()


def test_tc_tile_counter_reuse_and_concurrency(torch_cuda, poas):
    """The dynamic scheduler's self-resetting counters: more launches than
    the counter ring holds, both kernels interleaved, and two streams
    launching concurrently -- every result exact."""
    import oracle

    torch = torch_cuda
    m, n, k = 640, 768, 256
    A, B = oracle.fill_uniform(m, k, 41), oracle.fill_uniform(k, n, 42)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c1 = torch.full((m, n), float("nan"), device="cuda")
    c2 = torch.full((m, n), float("nan"), device="cuda")
    torch.cuda.synchronize()
    for i in range(300):  # ring of 256 counters wraps
        for st, c, ctas in ((s1, c1, 0), (s2, c2, 7 + (i % 5))):
            poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n,
                         num_ctas=ctas, stream=st.cuda_stream)
    torch.cuda.synchronize()
    for c in (c1, c2):
        assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL


def test_tc_wave_scheduler_survives_non_resident_workers(torch_cuda, poas, monkeypatch):
    """Wave mode with more persistent workers than SMs (the late ones are not
    resident until others exit): the per-wave barriers time out once and the
    kernel finishes with exact results instead of hanging."""
    import time

    import oracle

    torch = torch_cuda
    monkeypatch.setenv("POAS_TC_SCHED", "wave")
    m, n, k = 8192, 4096, 256  # 512 pair tiles; 400 CTAs = 200 pairs, 74 resident
    A, B = oracle.fill_uniform(m, k, 51), oracle.fill_uniform(k, n, 52)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    for ctas in (0, 400):
        c = torch.full((m, n), float("nan"), device="cuda")
        t0 = time.perf_counter()
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, num_ctas=ctas)
        torch.cuda.synchronize()
        assert time.perf_counter() - t0 < 5.0
        assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL, ctas


def _panel_major(torch, B16, panels):
    k, n = B16.shape
    np_ = n // panels
    return torch.stack([B16[:, p * np_:(p + 1) * np_] for p in range(panels)]).contiguous()


@pytest.mark.parametrize("variant", [None, "2cta512", "2cta512x2", "2cta256x2"])
@pytest.mark.parametrize("panels", [2, 4])
@pytest.mark.parametrize("shape", [(1000, 1024, 320), (300, 2048, 136)])
def test_tc_gemm_panels(torch_cuda, poas, monkeypatch, shape, panels, variant):
    """One launch over panel-major B (the layout a per-panel broadcast
    lands): tiles are ordered panel by panel and B is read through a 3-D
    tensor map; with readiness flags already set and without flags. With
    2cta512, panels that are whole 512-column tiles run the wide pair tile
    and the others the 256-wide one."""
    import oracle

    torch = torch_cuda
    if variant:
        monkeypatch.setenv("POAS_TC_KERNEL", variant)
    m, n, k = shape
    A, B = oracle.fill_uniform(m, k, 51), oracle.fill_uniform(k, n, 52)
    a = torch.from_numpy(A).cuda().bfloat16()
    bp = _panel_major(torch, torch.from_numpy(B).cuda().bfloat16(), panels)
    ref = oracle.gemm_rows_f64(A, B, 2)
    flags = torch.ones(panels, dtype=torch.int32, device="cuda")
    for fl in (None, flags.data_ptr()):
        for ctas in (0, 10):
            c = torch.full((m, n), float("nan"), device="cuda")
            poas.tc_gemm_panels(2, m, n, k, a.data_ptr(), k, bp.data_ptr(), n // panels, c.data_ptr(), n,
                                panels, flags=fl, epoch=1, num_ctas=ctas)
            torch.cuda.synchronize()
            assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL, (fl, ctas)
    from paper_2209_10245_b200 import PoasError

    with pytest.raises(PoasError):  # a panel narrower than a pair tile
        poas.tc_gemm_panels(2, m, 768, k, a.data_ptr(), k, bp.data_ptr(), 384, c.data_ptr(), n, 2)


@pytest.mark.parametrize("variant", ["2cta", "2cta512", "2cta512x2", "2cta256x2"])
def test_tc_gemm_panels_waits_for_flags(torch_cuda, poas, monkeypatch, variant):
    """The fused consumer: the GEMM is queued first with every flag clear;
    another stream delivers the panels later (a ~spin, then one flag per
    panel in order, each after the panel's bytes were written). The kernel
    must not read a panel before its flag: B is garbage until delivered."""
    import oracle

    torch = torch_cuda
    monkeypatch.setenv("POAS_TC_KERNEL", variant)
    m, n, k, panels = 2048, 2048, 512, 4
    A, B = oracle.fill_uniform(m, k, 61), oracle.fill_uniform(k, n, 62)
    a = torch.from_numpy(A).cuda().bfloat16()
    good = _panel_major(torch, torch.from_numpy(B).cuda().bfloat16(), panels)
    bp = torch.full_like(good, float("nan"))
    ref = oracle.gemm_rows_f64(A, B, 2)
    flags = torch.zeros(panels, dtype=torch.int32, device="cuda")
    c = torch.full((m, n), float("nan"), device="cuda")
    s_gemm, s_deliver = torch.cuda.Stream(), torch.cuda.Stream()
    # warm the delivery side first: a kernel's first launch may load its
    # module lazily, which waits for the device -- and the device would be
    # waiting (spinning) for this delivery
    scratch = torch.zeros(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s_deliver):
        torch.cuda._sleep(1)
        bp[0].copy_(good[0])
        bp[0].fill_(float("nan"))
        poas.signal_flag(scratch.data_ptr(), 1, s_deliver.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_gemm):
        e0.record()
        poas.tc_gemm_panels(2, m, n, k, a.data_ptr(), k, bp.data_ptr(), n // panels, c.data_ptr(), n,
                            panels, flags=flags.data_ptr(), epoch=7, num_ctas=64,
                            stream=s_gemm.cuda_stream)
        e1.record()
    with torch.cuda.stream(s_deliver):
        for p in range(panels):
            torch.cuda._sleep(2_000_000)  # ~1 ms
            bp[p].copy_(good[p])
            poas.signal_flag(flags[p:p + 1].data_ptr(), 7, s_deliver.cuda_stream)
    torch.cuda.synchronize()
    assert oracle.rel_frobenius(c.cpu().numpy(), ref) <= TOL
    assert e0.elapsed_time(e1) > 2.0  # it waited for the deliveries


def test_tc_variant_choice(torch_cuda, poas, monkeypatch):
    """256 x 512 pair tiles from two waves of them (and K >= 6144), 256 x 256
    pair tiles below, single-SM tiles when the grid of 128 x 128 tiles fits
    in one wave (128 x 64 when it fills at most half); the env override
    wins."""
    monkeypatch.delenv("POAS_TC_KERNEL", raising=False)
    assert poas.tc_kernel_name(16384, 16384, 16384) == "tc_gemm_2cta_kernel<512>"
    assert poas.tc_kernel_name(65536, 8192, 8192) == "tc_gemm_2cta_kernel<512>"
    assert poas.tc_kernel_name(8192, 8192, 8192) == "tc_gemm_2cta_kernel<512>"
    assert poas.tc_kernel_name(4096, 4096, 4096) == "tc_gemm_2cta_kernel<256>"
    assert poas.tc_kernel_name(1024, 1024, 1024) == "tc_gemm_kernel_n64"
    assert poas.tc_kernel_name(1536, 1536, 1536) == "tc_gemm_kernel_n128"
    assert poas.tc_kernel_name(2048, 2048, 2048) == "tc_gemm_2cta_kernel<256>"
    assert poas.tc_kernel_name(256, 4096, 16384) == "tc_gemm_kernel_n64"
    monkeypatch.setenv("POAS_TC_KERNEL", "2cta")
    assert poas.tc_kernel_name(1024, 1024, 1024) == "tc_gemm_2cta_kernel<256>"
    assert poas.tc_kernel_name(16384, 16384, 16384) == "tc_gemm_2cta_kernel<256>"
    monkeypatch.setenv("POAS_TC_KERNEL", "2cta512")
    assert poas.tc_kernel_name(1024, 1024, 1024) == "tc_gemm_2cta_kernel<512>"
    monkeypatch.setenv("POAS_TC_KERNEL", "2cta512x2")
    assert poas.tc_kernel_name(1024, 1024, 1024) == "tc_gemm_2cta_kernel<512,2>"
    monkeypatch.setenv("POAS_TC_KERNEL", "2cta256x2")
    assert poas.tc_kernel_name(1024, 1024, 1024) == "tc_gemm_2cta_kernel<256,2>"


@pytest.mark.parametrize("variant", ["2cta512", "2cta512x2", "2cta512:direct"])
@pytest.mark.parametrize("shape,ctas", [((2048, 4096, 2048), 4), ((1024, 2048, 64), 2),
                                        ((777, 1536, 4104), 8), ((4096, 1000, 192), 148),
                                        ((1300, 2560, 512), 12)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_tc_wide_pair_half_release(torch_cuda, poas, monkeypatch, shape, ctas, accumulate, variant):
    """256 x 512 pair tiles: the epilogue frees each 256-column half of the
    TMEM accumulator separately and the next tile's MMAs for half 1 trail
    half 0's by up to a ring of staged k-blocks. Many tiles per pair (long
    and short K -- one k-block: the end-of-tile catch-up), ragged N, and a
    budget of every SM; exact vs the oracle, plain and accumulating. The
    2cta512x2 clusters (two pairs sharing B by multicast) also run an odd
    number of 256-row tiles (a half-empty cluster tile) and budgets below
    one cluster (falls back to single pairs)."""
    import oracle

    torch = torch_cuda
    variant, _, epilogue = variant.partition(":")
    monkeypatch.setenv("POAS_TC_KERNEL", variant)
    if epilogue:
        monkeypatch.setenv("POAS_TC_EPILOGUE", epilogue)
    m, n, k = shape
    A, B = oracle.fill_uniform(m, k, 71), oracle.fill_uniform(k, n, 72)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    c = torch.full((m, n), 1.0 if accumulate else float("nan"), device="cuda")
    for _ in range(2):  # the second launch reuses the self-reset tile counter
        if accumulate:
            c.fill_(1.0)
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n,
                     accumulate=accumulate, num_ctas=ctas)
        torch.cuda.synchronize()
        got = c.cpu().numpy() - (1.0 if accumulate else 0.0)
        assert oracle.rel_frobenius(got, ref) <= TOL, (shape, ctas)


# (shape, SM budget) where the last wave of pair tiles is at most half a
# wave, so its tiles run as two K-halves (TcArgs::split_*): 1000^2 x 1000 on
# 5 pairs (16 tiles: 15 whole + 1 split), 1024^2 x 768 on 32 pairs (all 16
# tiles split: 32 halves), 4096^2 x 512 on the whole chip (256 tiles, the
# last 34 split on 74 pairs), and a ragged K tail (K = 1000: 16 k-blocks,
# the last one partial, in part 1; 24 tiles on 7 pairs).
_SPLIT_CASES = [((1000, 1000, 1000), 10), ((1024, 1024, 768), 64), ((4096, 4096, 512), 0),
                ((777, 1304, 1000), 14)]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["2cta", "2cta512"])
@pytest.mark.parametrize("accumulate", [False, True])
@pytest.mark.parametrize("case", _SPLIT_CASES)
def test_tc_last_wave_split(torch_cuda, poas, monkeypatch, variant, accumulate, case):
    """Last-wave K split: the split tiles' first K-half stores, the second
    add-reduces after the first's ready flag. C matches the oracle (plain and
    accumulating), equals itself bitwise over repeated launches (the ready
    flags and counters are left zero by every launch) and stays within the
    tolerance of the unsplit kernel (POAS_TC_SPLIT=0)."""
    import oracle

    torch = torch_cuda
    (m, n, k), ctas = case
    monkeypatch.setenv("POAS_TC_KERNEL", variant)
    monkeypatch.setenv("POAS_TC_SCHED", "dynamic")
    A, B = oracle.fill_uniform(m, k, 51), oracle.fill_uniform(k, n, 52)
    a = torch.from_numpy(A).cuda().bfloat16()
    b = torch.from_numpy(B).cuda().bfloat16()
    ref = oracle.gemm_rows_f64(A, B, 2)
    c0 = np.random.default_rng(5).uniform(-1, 1, (m, n)).astype(np.float32) if accumulate else None
    outs = []
    for split in ("1", "1", "1", "0"):
        monkeypatch.setenv("POAS_TC_SPLIT", split)
        c = torch.from_numpy(c0).cuda() if accumulate else torch.full((m, n), float("nan"), device="cuda")
        for _ in range(2 if split == "1" else 1):  # back-to-back launches on one stream
            if accumulate:
                c.copy_(torch.from_numpy(c0))
            poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n,
                         accumulate=accumulate, num_ctas=ctas)
        torch.cuda.synchronize()
        got = c.cpu().numpy()
        want = ref + (c0.astype(np.float64) if accumulate else 0)
        assert oracle.rel_frobenius(got, want) <= TOL, (variant, split, case)
        outs.append(got)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
