"""GPU: the tcgen05/TMEM/TMA implicit-GEMM conv kernel against a plain fp32
reference of the same op (torch on CPU, bf16-rounded operands).

Tolerance: the kernel accumulates in fp32 (TMEM) and rounds the epilogue to
bf16, so each element may differ from the fp32 reference by one bf16
rounding: |got - ref| <= 2^-7 * |ref| + 1e-3."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bf16_bits(x: torch.Tensor) -> np.ndarray:
    return x.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()


def run_gemm(ctx, A, Bw, N, Kc, ntaps, taps, bias, residual, relu, mode, H, W, M,
             rows_out, out_f32, BN, max_ctas=0, pair=0):
    a = bf16_bits(A)
    b = bf16_bits(Bw)
    res = None if residual is None else bf16_bits(residual)
    t = np.array(list(taps) + [0] * (9 - len(taps)), np.int32)
    bias = np.ascontiguousarray(bias, np.float32)
    out = np.zeros((rows_out, N), np.float32 if out_f32 else np.uint16)
    fn = ctx.L.cg_dbg_conv_gemm_pair if pair else ctx.L.cg_dbg_conv_gemm
    rc = fn(
        ctx.h, a.ctypes.data_as(C.c_void_p), A.shape[0], b.ctypes.data_as(C.c_void_p),
        N, Kc, ntaps, t.ctypes.data_as(C.c_void_p), bias.ctypes.data_as(C.c_void_p),
        None if res is None else res.ctypes.data_as(C.c_void_p), relu, mode, H, W, M,
        rows_out, out_f32, BN, out.ctypes.data_as(C.c_void_p), max_ctas)
    assert rc == 0, ctx.L.cg_last_error(ctx.h)
    if out_f32:
        return torch.from_numpy(out)
    return torch.from_numpy(out.view(np.int16)).view(torch.bfloat16).float()


def grid_rows(xq):
    """[NB, C, H, W] -> the kernels' shared-border zero grid as NHWC rows:
    per image H + 1 grid rows of W pixels + 1 zero column, grid row 0 zero
    (remap_row in csrc/gemm_sm100.cu). Returns (rows, pitch W + 1)."""
    NB, C, H, W = xq.shape
    z = torch.zeros(NB, H + 1, W + 1, C)
    z[:, 1:, :W, :] = xq.permute(0, 2, 3, 1)
    return z.reshape(-1, C), W + 1


def close(got, ref):
    err = (got - ref).abs()
    lim = 2.0 ** -7 * ref.abs() + 1e-3
    bad = (err > lim).sum().item()
    assert bad == 0, f"{bad} mismatches, max err {err.max().item()}"


def q(x):
    return x.to(torch.bfloat16).float()


@pytest.mark.parametrize("M,N,Kc,BN,relu,max_ctas", [
    (300, 128, 256, 128, 1, 0), (128, 64, 64, 64, 0, 0), (1000, 512, 128, 256, 1, 0),
    (2048, 256, 512, 128, 0, 3), (4096, 64, 576, 64, 1, 5), (777, 256, 64, 256, 0, 2),
    # N not a multiple of the tile: the last tile's upper 64-column block /
    # 32-column half is clipped (bulk store) or skipped (bias, remap stores)
    (500, 96, 128, 64, 1, 0), (600, 160, 192, 128, 1, 0), (333, 320, 64, 256, 0, 0)])
def test_gemm_1x1(ctx, M, N, Kc, BN, relu, max_ctas):
    g = torch.Generator().manual_seed(M + N)
    A = torch.rand(M, Kc, generator=g) * 2 - 1
    Bw = torch.rand(N, Kc, generator=g) * 2 - 1
    bias = torch.rand(N, generator=g) - 0.5
    got = run_gemm(ctx, A, Bw, N, Kc, 1, [0], bias, None, relu, 0, 0, 0, M, M, 0, BN, max_ctas)
    ref = q(A) @ q(Bw).T + bias
    if relu:
        ref = ref.clamp_min(0)
    close(got, ref)


def test_gemm_residual_and_f32_tail(ctx):
    g = torch.Generator().manual_seed(3)
    M, N, Kc = 513, 256, 192
    A = torch.rand(M, Kc, generator=g) * 2 - 1
    Bw = torch.rand(N, Kc, generator=g) * 2 - 1
    R = torch.rand(M, N, generator=g) * 2 - 1
    bias = torch.rand(N, generator=g) - 0.5
    got = run_gemm(ctx, A, Bw, N, Kc, 1, [0], bias, R, 1, 0, 0, 0, M, M, 0, 128)
    close(got, (q(A) @ q(Bw).T + bias + q(R)).clamp_min(0))
    # FC shape: N = 1000 (not a multiple of the tile), f32 logits
    N = 1000
    Bw = torch.rand(N, Kc, generator=g) * 2 - 1
    bias = torch.rand(N, generator=g) - 0.5
    got = run_gemm(ctx, A[:128], Bw, N, Kc, 1, [0], bias, None, 0, 0, 0, 0, 128, 128, 1, 128)
    ref = q(A[:128]) @ q(Bw).T + bias
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,N,Kc,BN", [(700, 512, 640, 256), (1500, 256, 512, 128),
                                        (333, 128, 1024, 64), (2000, 1024, 256, 256),
                                        (900, 96, 256, 64), (700, 320, 128, 256)])
def test_gemm_residual_ring_configs(ctx, M, N, Kc, BN):
    """Both residual-ring layouts (deep ring for short K, more mainloop
    stages for K >= 512) over ragged tails."""
    g = torch.Generator().manual_seed(M * 3 + Kc)
    A = torch.rand(M, Kc, generator=g) * 2 - 1
    Bw = (torch.rand(N, Kc, generator=g) * 2 - 1) / 8
    R = torch.rand(M, N, generator=g) * 2 - 1
    bias = torch.rand(N, generator=g) - 0.5
    got = run_gemm(ctx, A, Bw, N, Kc, 1, [0], bias, R, 1, 0, 0, 0, M, M, 0, BN)
    close(got, (q(A) @ q(Bw).T + bias + q(R)).clamp_min(0))


@pytest.mark.parametrize("M,N,Kc,res,relu,max_ctas,out_f32", [
    (300, 256, 256, 0, 1, 0, 0), (777, 512, 192, 1, 1, 0, 0), (2048, 1024, 512, 1, 0, 6, 0),
    (128, 256, 64, 1, 1, 0, 0), (5000, 2048, 128, 0, 1, 0, 0), (256, 1000, 128, 0, 0, 0, 1)])
def test_gemm_pair(ctx, M, N, Kc, res, relu, max_ctas, out_f32):
    """SM-pair (cta_group::2) 256 x 256 tiles: ragged row tails (a peer CTA
    with no rows), the residual ring, a capped grid, f32 logits (FC shape)."""
    g = torch.Generator().manual_seed(M + 7 * N)
    A = torch.rand(M, Kc, generator=g) * 2 - 1
    Bw = torch.rand(N, Kc, generator=g) * 2 - 1
    R = torch.rand(M, N, generator=g) * 2 - 1 if res else None
    bias = torch.rand(N, generator=g) - 0.5
    got = run_gemm(ctx, A, Bw, N, Kc, 1, [0], bias, R, relu, 0, 0, 0, M, M, out_f32, 256,
                   max_ctas, pair=1)
    ref = q(A) @ q(Bw).T + bias
    if res:
        ref = ref + q(R)
    if relu:
        ref = ref.clamp_min(0)
    if out_f32:
        assert torch.allclose(got, ref, rtol=1e-4, atol=1e-3)
    else:
        close(got, ref)


def test_gemm_pair_taps_remap(ctx):
    """SM pairs over 9 row-shifted taps with a row remap (PadToCompact)."""
    NB, H, C, Cout = 2, 14, 64, 256
    W = H
    g = torch.Generator().manual_seed(11)
    x = torch.rand(NB, C, H, W, generator=g) * 2 - 1
    w = (torch.rand(Cout, C, 3, 3, generator=g) * 2 - 1) / 3
    bias = torch.rand(Cout, generator=g) - 0.5
    A, Wp = grid_rows(q(x))
    taps = [(dr - 1) * Wp + (ds - 1) for dr in range(3) for ds in range(3)]
    Bw = q(w).permute(0, 2, 3, 1).reshape(Cout, 9 * C)
    M = A.shape[0]
    got = run_gemm(ctx, A, Bw, Cout, C, 9, taps, bias, None, 1, 1, H, W, M, NB * H * W, 0, 256,
                   pair=1)
    ref = torch.nn.functional.conv2d(q(x), q(w), bias, padding=1).clamp_min(0)
    close(got, ref.permute(0, 2, 3, 1).reshape(-1, Cout))


@pytest.mark.parametrize("NB,H,C,Cout,BN", [(3, 7, 64, 128, 128), (2, 14, 128, 64, 64),
                                            (2, 28, 64, 256, 256), (2, 14, 64, 96, 64),
                                            (2, 7, 128, 160, 128)])
def test_conv3x3_padded_grid(ctx, NB, H, C, Cout, BN):
    """3x3/stride-1/pad-1 conv as 9 row-shifted taps over the zero-bordered
    grid (row mode PadToCompact) == torch conv2d."""
    W = H
    g = torch.Generator().manual_seed(H * C)
    x = torch.rand(NB, C, H, W, generator=g) * 2 - 1
    w = (torch.rand(Cout, C, 3, 3, generator=g) * 2 - 1) / 3
    bias = torch.rand(Cout, generator=g) - 0.5
    A, Wp = grid_rows(q(x))                                     # zero-bordered NHWC rows
    taps = [(dr - 1) * Wp + (ds - 1) for dr in range(3) for ds in range(3)]
    Bw = q(w).permute(0, 2, 3, 1).reshape(Cout, 9 * C)          # [Cout, (dr,ds,c)]
    M = A.shape[0]
    got = run_gemm(ctx, A, Bw, Cout, C, 9, taps, bias, None, 1, 1, H, W, M, NB * H * W, 0, BN)
    ref = torch.nn.functional.conv2d(q(x), q(w), bias, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    close(got, ref)


def run_halo(ctx, A, Bw, N, Kc, taps, bias, H, W, M, rows_out, BN, halo_lo, pair=False):
    a = bf16_bits(A)
    b = bf16_bits(Bw)
    t = np.array(list(taps), np.int32)
    bias = np.ascontiguousarray(bias, np.float32)
    out = np.zeros((rows_out, N), np.uint16)
    fn = ctx.L.cg_dbg_conv_gemm_halo_pair if pair else ctx.L.cg_dbg_conv_gemm_halo
    rc = fn(
        ctx.h, a.ctypes.data_as(C.c_void_p), A.shape[0], b.ctypes.data_as(C.c_void_p), N, Kc,
        9, t.ctypes.data_as(C.c_void_p), bias.ctypes.data_as(C.c_void_p), 1, 1, H, W, M,
        rows_out, BN, out.ctypes.data_as(C.c_void_p), halo_lo)
    assert rc == 0, ctx.L.cg_last_error(ctx.h)
    return torch.from_numpy(out.view(np.int16)).view(torch.bfloat16).float()


@pytest.mark.parametrize("NB,H,C,Cout,BN", [(3, 7, 64, 128, 128), (2, 14, 128, 64, 64),
                                            (2, 28, 64, 256, 256), (2, 56, 64, 64, 64),
                                            # wide halos: 2 / 3 stacked boxes per slot
                                            (1, 112, 64, 64, 64), (1, 112, 128, 128, 128),
                                            (1, 224, 64, 64, 64)])
def test_conv3x3_halo(ctx, NB, H, C, Cout, BN):
    """Halo mode: one (128 + 2*(W+2))-row box per channel block feeds all 9
    taps (MMA descriptors at arbitrary row offsets inside the 128B-swizzled
    halo) == torch conv2d. Halos wider than 256 rows arrive as stacked boxes
    (ConvGemmArgs::halo_sub) in one slot."""
    W = H
    g = torch.Generator().manual_seed(H * C + 1)
    x = torch.rand(NB, C, H, W, generator=g) * 2 - 1
    w = (torch.rand(Cout, C, 3, 3, generator=g) * 2 - 1) / 3
    bias = torch.rand(Cout, generator=g) - 0.5
    A, Wp = grid_rows(q(x))
    taps = [(dr - 1) * Wp + (ds - 1) for dr in range(3) for ds in range(3)]
    Bw = q(w).permute(0, 2, 3, 1).reshape(Cout, 9 * C)
    M = A.shape[0]
    ref = torch.nn.functional.conv2d(q(x), q(w), bias, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    got = run_halo(ctx, A, Bw, Cout, C, taps, bias, H, W, M, NB * H * W, BN, Wp + 1)
    close(got, ref)


def test_compact_to_padded_interior(ctx):
    NB, H, C, Cout = 2, 7, 64, 64
    W, Wp = H, H + 1
    g = torch.Generator().manual_seed(9)
    A = torch.rand(NB * H * W, C, generator=g) * 2 - 1
    Bw = torch.rand(Cout, C, generator=g) * 2 - 1
    bias = torch.zeros(Cout)
    rows_out = NB * (H + 1) * Wp
    got = run_gemm(ctx, A, Bw, Cout, C, 1, [0], bias, None, 1, 2, H, W, NB * H * W,
                   rows_out, 0, 64)
    ref = (q(A) @ q(Bw).T).clamp_min(0).reshape(NB, H, W, Cout)
    gp = got.reshape(NB, H + 1, Wp, Cout)
    close(gp[:, 1:, :W], ref)
    # the shared zero row / column stay zero
    assert gp[:, 0].abs().sum() == 0 and gp[:, :, W].abs().sum() == 0


@pytest.mark.parametrize("BN", [64, 128, 256])
def test_gemm_many_tiles_per_cta_tma_store(ctx, BN):
    """Many tiles per CTA through the TMA-store epilogue (staging buffers are
    reused across tiles): catches write-after-read races on smem staging."""
    g = torch.Generator().manual_seed(BN)
    M, N, Kc = 128 * 40, 256, 64
    A = torch.rand(M, Kc, generator=g) * 2 - 1
    Bw = torch.rand(N, Kc, generator=g) * 2 - 1
    R = torch.rand(M, N, generator=g) * 2 - 1
    bias = torch.rand(N, generator=g) - 0.5
    for res in (None, R):
        got = run_gemm(ctx, A, Bw, N, Kc, 1, [0], bias, res, 1, 0, 0, 0, M, M, 0, BN, max_ctas=2)
        ref = q(A) @ q(Bw).T + bias + (0 if res is None else q(res))
        close(got, ref.clamp_min(0))


@pytest.mark.parametrize("NB,H,C,Cout", [(3, 7, 64, 128), (2, 28, 128, 128), (1, 14, 256, 512)])
def test_conv3x3_halo_sm_pair(ctx, NB, H, C, Cout):
    """SM-pair halo mode (cluster of 2, cta_group::2 M=256 MMAs over both
    CTAs' shared memory, weights split by N across the pair) == torch."""
    W = H
    g = torch.Generator().manual_seed(H * C + 7)
    x = torch.rand(NB, C, H, W, generator=g) * 2 - 1
    w = (torch.rand(Cout, C, 3, 3, generator=g) * 2 - 1) / 3
    bias = torch.rand(Cout, generator=g) - 0.5
    A, Wp = grid_rows(q(x))
    taps = [(dr - 1) * Wp + (ds - 1) for dr in range(3) for ds in range(3)]
    Bw = q(w).permute(0, 2, 3, 1).reshape(Cout, 9 * C)
    M = A.shape[0]
    ref = torch.nn.functional.conv2d(q(x), q(w), bias, padding=1).clamp_min(0)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Cout)
    got = run_halo(ctx, A, Bw, Cout, C, taps, bias, H, W, M, NB * H * W, 128, Wp + 1, pair=True)
    close(got, ref)
