"""Elementwise parity at the BASELINE sizes the bench runs.

The kernels' outputs are compared, full rows at a time, with the fp64 CPU
oracle (oracle/gemm_oracle.c: the operands regenerated from the reference's
counter-based stream, rounded to the unit's precision, fp64 accumulation)
on 64 sampled rows: the first and last, 128/256-row tile boundaries spread
over M, and random rows (oracle.sampled_rows).

  C3   16384^3   bf16 tensor unit alone (pair kernel, dynamic scheduler)
                 and the POAS plan through the executor (resident operands)
  C5   32768^3   the default path there (wave tile scheduler, >= 2^44 MACs)
  C4   65536 x 8192 x 8192 (one GPU's view of the row-sharded shape)

Tolerance (stated): relative Frobenius over the sampled rows <= 2e-5 for
K <= 16384, and 2e-5 * K/16384 beyond (fp32 accumulation on
the tensor pipe loses accuracy ~linearly in K); in every case also <= 1.5x
cuBLAS's error on the same rows and inputs.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 20261017


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def tol_for(k: int) -> float:
    return 2e-5 * max(1.0, k / 16384.0)


def _operands(torch, poas, m, n, k):
    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")
    a = torch.empty(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(k, n, device="cuda", dtype=torch.bfloat16)
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), k, m, k, 0, 0, k, sa)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, k, n, 0, 0, n, sb)
    return a, b, sa, sb


def _check_rows(torch, C, a, b, rows, sa, sb, n, k, label):
    import oracle

    ref = oracle.full_size_rows_f64(rows, n, k, sa, sb, 2)
    idx = torch.from_numpy(rows).cuda()
    got = C.index_select(0, idx).cpu().numpy()
    err = oracle.rel_frobenius(got, ref)
    lib = torch.mm(a.index_select(0, idx), b, out_dtype=torch.float32).cpu().numpy()
    err_lib = oracle.rel_frobenius(lib, ref)
    print(f"{label}: sampled-row rel err {err:.3e} (cuBLAS {err_lib:.3e}), tol {tol_for(k):.1e}")
    assert np.isfinite(got).all(), label
    assert err <= tol_for(k), (label, err, err_lib)
    assert err <= 1.5 * err_lib + 1e-7, (label, err, err_lib)
    return err


@pytest.mark.parametrize("m,n,k", [(16384, 16384, 16384), (32768, 32768, 32768), (65536, 8192, 8192)])
def test_tc_full_size_sampled_rows(torch_cuda, poas, m, n, k):
    """The tensor kernel on its default path at each BASELINE size."""
    import oracle

    torch = torch_cuda
    a, b, sa, sb = _operands(torch, poas, m, n, k)
    C = torch.full((m, n), float("nan"), device="cuda")
    poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, C.data_ptr(), n)
    torch.cuda.synchronize()
    label = f"{m}x{n}x{k} {poas.tc_kernel_name(m, n, k)}/{poas.tc_scheduler_name(m, n, k)}"
    rows = oracle.sampled_rows(m)
    _check_rows(torch, C, a, b, rows, sa, sb, n, k, label)
    # against the unrounded fp32 inputs (BASELINE.md section 3, bf16 <= 8e-3)
    got = C.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    err_exact = oracle.rel_frobenius(got, oracle.full_size_rows_f64(rows, n, k, sa, sb, 0))
    print(f"{label}: vs unrounded inputs {err_exact:.3e}")
    assert err_exact <= 8e-3, err_exact


def test_c2_fp16_tensor_full_size_sampled_rows(torch_cuda, poas):
    """C2's tensor share: fp16 operands at 8192^3 on the default (256 x 512
    pair-tile) kernel, sampled rows vs the oracle in fp16 rounding."""
    import oracle

    torch = torch_cuda
    n = k = m = 8192
    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")
    a32 = torch.empty(m, k, device="cuda")
    b32 = torch.empty(k, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_F32, a32.data_ptr(), k, m, k, 0, 0, k, sa)
    poas.fill_uniform(poas.DTYPE_F32, b32.data_ptr(), n, k, n, 0, 0, n, sb)
    a, b = a32.half(), b32.half()
    C = torch.full((m, n), float("nan"), device="cuda")
    poas.tc_gemm(poas.DTYPE_F16, m, n, k, a.data_ptr(), k, b.data_ptr(), n, C.data_ptr(), n)
    torch.cuda.synchronize()
    rows = oracle.sampled_rows(m)
    ref = oracle.full_size_rows_f64(rows, n, k, sa, sb, 1)
    got = C.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    err = oracle.rel_frobenius(got, ref)
    exact = oracle.full_size_rows_f64(rows, n, k, sa, sb, 0)  # unrounded fp32 inputs
    err_exact = oracle.rel_frobenius(got, exact)
    print(f"8192^3 fp16 {poas.tc_kernel_name(m, n, k)}: sampled-row rel err {err:.3e} "
          f"(vs unrounded inputs {err_exact:.3e})")
    assert poas.tc_kernel_name(m, n, k) == "tc_gemm_2cta_kernel<512>"
    assert np.isfinite(got).all() and err <= tol_for(k), err
    assert err_exact <= 2e-3, err_exact


def test_c3_poas_plan_full_size_sampled_rows(torch_cuda, poas):
    """C3 through the product path the bench times: profile the bench's two
    units, plan (best-subset), execute with resident operands; every sampled
    row of C checked against the oracle in its unit's operand precision."""
    import oracle

    torch = torch_cuda
    n = k = m = 16384
    units = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=8192-16384;"
             "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048")
    profile = poas.profile_machine(units, "probes=4,repetitions=2,bandwidth_payload=67108864", True)
    sched_text = poas.plan_policy(profile, m, n, k, "best-subset")
    sched = json.loads(sched_text)
    a, b, sa, sb = _operands(torch, poas, m, n, k)
    a32 = torch.empty(m, k, device="cuda")
    b32 = torch.empty(k, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_F32, a32.data_ptr(), k, m, k, 0, 0, k, sa)
    poas.fill_uniform(poas.DTYPE_F32, b32.data_ptr(), n, k, n, 0, 0, n, sb)
    C = torch.full((m, n), float("nan"), device="cuda")
    io = poas.GemmIO(m=m, n=n, k=k, a_dev=a32.data_ptr(), lda_dev=k, b_dev=b32.data_ptr(), ldb_dev=n,
                     a16_dev=a.data_ptr(), lda16_dev=k, b16_dev=b.data_ptr(), ldb16_dev=n,
                     c_dev=C.data_ptr(), ldc_dev=n, resident=1)
    poas.Executor(units).execute(sched_text, io, 1)
    torch.cuda.synchronize()
    rows = oracle.sampled_rows(m)
    r0 = 0
    for d in sched["devices"]:
        sel = rows[(rows >= r0) & (rows < r0 + d["rows"])]
        if len(sel):
            mode = 2 if d["id"] == "gpu0.tc" else 0
            ref = oracle.full_size_rows_f64(sel, n, k, sa, sb, mode)
            idx = torch.from_numpy(sel).cuda()
            err = oracle.rel_frobenius(C.index_select(0, idx).cpu().numpy(), ref)
            assert err <= tol_for(k), (d["id"], err)
        r0 += d["rows"]
    assert r0 == m
