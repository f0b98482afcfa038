"""Random-init kernel traces of the BASELINE.json model configs, as scenario
kernels (the reference's kernel records -- blocks, block_us, s, occ,
sim.cpp:86-156 / workload.hpp:38-44 -- plus the B200 "body" extension that
the reference ignores). Every kernel is one tenant launch; its blocks are
the body's real grid:

  conv_bf16  NHWC implicit GEMM (TMA im2col), 256 pixels x 256 channels per block
  gemm_bf16  256 x 256 output tile per block
  gemv_bf16  256 rows of W per block (x split-K)
  stream     HBM-bound elementwise (norms, activations, residuals, pooling,
             softmax, attention over the KV cache, optimizer), sized by the
             tensor bytes it moves

Each layer has its own workspace id, so each layer's weights are distinct
buffers (decode streams 15 GB of Llama-3-8B weights per token, as the real
model does). block_us / s are first estimates for the reference's timing
model (replay); the live scheduler's predictor learns measured latencies.

  resnet50_infer(batch)   ResNet-50 forward at 224 x 224   (configs #2, #3)
  bert_base_infer(batch)  BERT-base, seq 128               (config #2)
  llama3_8b_decode(ctx)   Llama-3-8B, one token at batch 1 (config #3)
  resnet50_train(batch)   ResNet-50 forward + backward + SGD (config #3)
"""
from __future__ import annotations

import math

TPC_TFLOPS = 1650.0 / 74      # measured bf16 peak per TPC
TPC_GBS = 6550.0 / 74         # measured HBM bandwidth per TPC
STREAM_WORDS = 16384          # u32 words per STREAM block (64 KiB in, 64 KiB out)


def n_tile(cols: int) -> int:
    """UMMA N of a pair tile over `cols` output columns (dispatcher.cu
    narrow_tile): narrow outputs do not compute padding columns."""
    return 64 if cols <= 64 else 128 if cols <= 128 else 256


def conv_blocks(n, h, w, c, k, r, s, pad, stride) -> tuple[int, int, int]:
    """Grid of gpuos_dev_conv_desc (conv_body.cuh): (blocks, P, Q) -- pair
    tiles of 256 consecutive output pixels (TMA im2col) x n_tile(k) channels."""
    P = (h + 2 * pad - r) // stride + 1
    Q = (w + 2 * pad - s) // stride + 1
    return math.ceil(n * P * Q / 256) * math.ceil(k / n_tile(k)), P, Q


def gemm_splits(k, splits) -> int:
    """Effective K splits of gpuos_dev_gemm_desc_splitk (every split non-empty)."""
    nk = math.ceil(k / 64)
    per = math.ceil(nk / max(1, min(splits, nk)))
    return math.ceil(nk / per)


def gemm_blocks(m, n, k, splits=1) -> int:
    return math.ceil(m / 256) * math.ceil(n / n_tile(n)) * gemm_splits(k, splits)


def wgrad_splits(m, n, k, target=296) -> int:
    """Split-K for a weight gradient (few output tiles, K = n P Q): enough
    splits for `target` blocks (two waves of the 148 worker pairs), each
    split at least 32 K steps of 64."""
    tiles = math.ceil(m / 256) * math.ceil(n / n_tile(n))
    return max(1, min(math.ceil(target / tiles), math.ceil(k / 64) // 32))


def gemv_blocks(n, k, splits) -> int:
    nk = math.ceil(k / 64)
    per = math.ceil(nk / max(1, splits))
    return math.ceil(n / 256) * math.ceil(nk / per)


class Builder:
    """Accumulates kernels; `ws` hands out a fresh workspace id per layer."""

    def __init__(self, ws_base: int):
        self.kernels: list[dict] = []
        self.ws = ws_base
        self.stream_ws = ws_base + 99_000  # one buffer pair for all elementwise kernels

    def _next(self) -> int:
        self.ws += 1
        return self.ws

    def conv(self, n, h, w, c, k, r, s, pad, stride) -> tuple[int, int]:
        blocks, P, Q = conv_blocks(n, h, w, c, k, r, s, pad, stride)
        cb = math.ceil(c / 64) * 64
        tile_flops = 2.0 * 256 * n_tile(k) * r * s * cb
        self.kernels.append({
            "blocks": blocks, "block_us": round(tile_flops / (TPC_TFLOPS * 1e6), 3), "s": 0.9, "occ": 2,
            "body": {"kind": "conv_bf16", "ws": self._next(), "p": [n, h, w, c, k, r, s, pad, stride]}})
        return P, Q

    def gemm(self, m, n, k, splits=1) -> None:
        sp = gemm_splits(k, splits)
        self.kernels.append({
            "blocks": gemm_blocks(m, n, k, sp),
            "block_us": round(2.0 * 256 * n_tile(n) * k / sp / (TPC_TFLOPS * 1e6), 3), "s": 0.9, "occ": 2,
            "body": {"kind": "gemm_bf16", "ws": self._next(), "p": [m, n, k] + ([sp] if sp > 1 else [])}})

    def gemv(self, n, k, splits=1) -> None:
        """occ 1: HBM-bound, so the occupancy filter (blocks / occ TPCs at
        most) lets it spread over every TPC rather than pack two per TPC."""
        blocks = gemv_blocks(n, k, splits)
        per_block = n * k * 2 / blocks
        self.kernels.append({
            "blocks": blocks, "block_us": round(per_block / (TPC_GBS * 1e3), 3), "s": 0.2, "occ": 1,
            "body": {"kind": "gemv_bf16", "ws": self._next(), "p": [n, k, splits]}})

    def rmsnorm(self, rows, d) -> None:
        """RMSNorm as the tenant body rmsnorm_bf16 (csrc/bodies): one row per
        block, 256 threads, HBM-bound (x and y: 4 d bytes per row)."""
        self.kernels.append({
            "blocks": rows, "block_us": round(max(1.0, 4.0 * d / (TPC_GBS / 4 * 1e3)), 3), "s": 0.2, "occ": 4,
            "body": {"kind": "rmsnorm_bf16", "ws": self._next(), "p": [rows, d]}})

    def silu_mul(self, n, chunk=2048) -> None:
        """SiLU(gate) * up as the tenant body silu_mul_bf16: `chunk` elements
        per block (6 bytes each: gate, up, out)."""
        self.kernels.append({
            "blocks": -(-n // chunk), "block_us": round(max(1.0, 6.0 * chunk / (TPC_GBS / 4 * 1e3)), 3),
            "s": 0.2, "occ": 4, "body": {"kind": "silu_mul_bf16", "ws": self._next(), "p": [n, chunk]}})

    def attention(self, ctx, chunk=32) -> None:
        """Decode GQA attention (32 query / 8 KV heads of 128, RoPE on the
        query) over a `ctx`-long KV cache as the tenant body attn_decode_bf16:
        block = (context chunk, KV head), chunks merged by the head's last
        block. occ 2: the planner spreads its 256 blocks over every TPC
        (stacked with training 16.0 us vs 17.6 us at occ 4 on 64 TPCs)."""
        blocks = -(-ctx // chunk) * 8
        self.kernels.append({
            "blocks": blocks, "block_us": round(max(1.0, 4.0 * chunk * 128 / (TPC_GBS / 4 * 1e3)), 3),
            "s": 0.2, "occ": 2, "body": {"kind": "attn_decode_bf16", "ws": self._next(), "p": [ctx, chunk]}})

    def stream(self, nbytes) -> None:
        """Elementwise kernel moving `nbytes` (read + written): blocks of at
        most STREAM_WORDS u32, sized (in 1 KiB steps) to the bytes moved, so
        a 16 KB RMSNorm is one 16 KB block, not a 128 KB one."""
        blocks = max(1, math.ceil(nbytes / (8 * STREAM_WORDS)))
        words = min(STREAM_WORDS, max(256, math.ceil(nbytes / (8 * blocks) / 256) * 256))
        self.kernels.append({
            "blocks": blocks, "block_us": round(8 * words / (TPC_GBS / 4 * 1e3), 3), "s": 0.2, "occ": 4,
            "body": {"kind": "stream", "ws": self.stream_ws, "p": [words, 0, 256]}})


RESNET_STAGES = [(3, 64, 256, 1), (4, 128, 512, 2), (6, 256, 1024, 2), (3, 512, 2048, 2)]


def _resnet_forward(b: Builder, n: int) -> list[tuple]:
    """Forward pass; returns the conv shapes (for the backward pass)."""
    convs = []

    def conv(*a):
        convs.append(a)
        return b.conv(*a)

    h = conv(n, 224, 224, 8, 64, 7, 7, 3, 2)[0]         # stem, 3 channels padded to 8
    b.stream(n * 112 * 112 * 64 * 2 * 2)                # BN + ReLU
    b.stream(n * (112 * 112 + 56 * 56) * 64 * 2)         # max pool 3x3/2
    h, c = 56, 64
    for blocks, mid, out, stride in RESNET_STAGES:
        for i in range(blocks):
            st = stride if i == 0 else 1
            conv(n, h, h, c, mid, 1, 1, 0, 1)
            ho = conv(n, h, h, mid, mid, 3, 3, 1, st)[0]
            conv(n, ho, ho, mid, out, 1, 1, 0, 1)
            if i == 0:
                conv(n, h, h, c, out, 1, 1, 0, st)       # downsample
            b.stream(n * ho * ho * out * 2 * 3)          # residual add + ReLU
            h, c = ho, out
    b.stream(n * 7 * 7 * 2048 * 2)                       # global average pool
    return convs


def resnet50_infer(batch: int = 1, ws_base: int = 0) -> list[dict]:
    b = Builder(ws_base)
    _resnet_forward(b, batch)
    if batch == 1:
        b.gemv(1000, 2048)                               # classifier
    else:
        b.gemm(batch, 1000, 2048)
    return b.kernels


def resnet50_train(batch: int = 64, ws_base: int = 0) -> list[dict]:
    """Forward, backward (for every conv: data-gradient conv of the same
    FLOPs and weight-gradient GEMM reduced over n p q), ReLU/BN backward
    elementwise, and an SGD-momentum update over 25.6 M fp32 params.

    The weight gradient dW[k, r s c] = dY^T . X_col has few output tiles and
    a K of n P Q (up to 800 K at batch 64): it is computed transposed,
    dW^T[r s c, k] (M = r s c, N = k: a 64-wide UMMA N for k = 64), with
    split-K over n P Q -- as cuDNN does -- so it spreads over the TPCs
    instead of 13 tiles running 8 ms each on 7 TPCs (round-2 measurement,
    tools/train_breakdown.py)."""
    b = Builder(ws_base)
    convs = _resnet_forward(b, batch)
    b.gemm(batch, 1000, 2048)
    b.gemm(1000, 2048, batch if batch % 8 == 0 else 8)   # classifier weight gradient
    for (n, h, w, c, k, r, s, pad, stride) in reversed(convs):
        P = (h + 2 * pad - r) // stride + 1
        if c >= 64:                                      # no data gradient for the stem input
            b.conv(n, P, P, k, c, r, s, (r - 1) // 2, 1)  # dgrad (same FLOPs as forward)
        m_w, n_w, k_w = r * s * c, k, n * P * P              # (stem: its 8 padded input channels)
        b.gemm(m_w, n_w, k_w, wgrad_splits(m_w, n_w, k_w))    # wgrad (transposed, split-K)
        b.stream(n * P * P * k * 2 * 3)                  # BN / ReLU backward
    b.stream(25_600_000 * 4 * 5)                         # SGD with momentum: w, g, m read; w, m written
    return b.kernels


def bert_base_infer(batch: int = 8, seq: int = 128, ws_base: int = 0) -> list[dict]:
    b = Builder(ws_base)
    t = batch * seq
    d, heads, ffn = 768, 12, 3072
    b.stream(t * d * 2 * 3)                              # embeddings + LayerNorm
    for _ in range(12):
        b.gemm(t, 3 * d, d)                              # QKV projection
        b.gemm(batch * heads * seq, seq, d // heads)     # scores (per-head GEMMs as one of equal FLOPs)
        b.stream(batch * heads * seq * seq * 2 * 2)      # softmax
        b.gemm(batch * heads * seq, d // heads, seq)     # context
        b.gemm(t, d, d)                                  # output projection
        b.stream(t * d * 2 * 3)                          # residual + LayerNorm
        b.gemm(t, ffn, d)                                # FFN up
        b.stream(t * ffn * 2 * 2)                        # GELU
        b.gemm(t, d, ffn)                                # FFN down
        b.stream(t * d * 2 * 3)                          # residual + LayerNorm
    return b.kernels


def llama3_8b_decode(context: int = 1024, ws_base: int = 0,
                     splits: tuple = (3, 4, 1, 4), attention: bool = False) -> list[dict]:
    """One token: 32 layers of RMSNorm, QKV / O / gate-up / down GEMVs (split-K
    so every TPC streams weights), attention over a `context`-long KV cache
    (8 KV heads x 128), SiLU-mul; then the final norm and the LM head.
    `splits` (QKV, O, gate-up, down) size each GEMV to about one wave of one
    worker pair per TPC (72 / 64 / 112 / 64 blocks): stacked with a
    best-effort tenant, whose tiles hold the TPCs' other pairs, a decode GEMV
    still runs in one wave. Sized to both pairs (6, 8, 1, 9: 144 / 128 / 112
    / 144 blocks) decode alone is 6 % faster but stacked 24 % slower, as the
    second wave waits for best-effort tiles (tools/hybrid_breakdown.py: QKV
    17.7 us alone / 29.6 us stacked vs 20.1 / 21.8; token p50 4.71 / 6.13 ms
    vs 5.02 / 5.73 ms).
    `attention`: run decode attention as the tenant body attn_decode_bf16
    (real GQA + RoPE, value-checked) instead of a STREAM kernel moving the
    same bytes. Measured (tools/hybrid_breakdown.py): the body takes 14.6 us
    alone / 21 us stacked against 8 us for the byte-equivalent stream (256
    blocks: wake-up and claim skew, the chunk merge's extra round trips), and
    config #3's decode p99 goes 1.15x -> 1.28x alone; the config keeps the
    stream by default and the bench reports the real-attention variant
    beside it."""
    b = Builder(ws_base)
    d, kv, ffn, vocab = 4096, 1024, 14336, 128256
    for _ in range(32):
        b.rmsnorm(1, d)                                  # RMSNorm (tenant body)
        b.gemv(d + 2 * kv, d, splits[0])                 # QKV (72 blocks)
        if attention:
            b.attention(context)                         # RoPE + attention over the KV cache (tenant body)
        else:
            b.stream(context * kv * 2 * 2 + d * 2 * 2)   # ... as a byte-equivalent STREAM kernel
        b.gemv(d, d, splits[1])                          # output projection (64 blocks)
        b.rmsnorm(1, d)                                  # residual + RMSNorm (tenant body)
        b.gemv(2 * ffn, d, splits[2])                    # gate + up (112 blocks)
        b.silu_mul(ffn)                                  # SiLU(gate) * up (tenant body, 7 blocks)
        b.gemv(d, ffn, splits[3])                        # down projection (64 blocks)
    b.rmsnorm(1, d)                                      # final norm
    b.gemv(vocab, d, 1)                                  # LM head
    return b.kernels


def summary(kernels: list[dict]) -> dict:
    """Kernel count, blocks and algorithmic work of a trace."""
    flops = nbytes = 0.0
    for k in kernels:
        body, p = k["body"], k["body"]["p"]
        if body["kind"] == "gemm_bf16":
            flops += 2.0 * p[0] * p[1] * p[2]
            nbytes += 2.0 * (p[0] * p[2] + p[1] * p[2] + p[0] * p[1])
        elif body["kind"] == "conv_bf16":
            n, h, w, c, kk, r, s, pad, st = p
            P = (h + 2 * pad - r) // st + 1
            Q = (w + 2 * pad - s) // st + 1
            flops += 2.0 * n * P * Q * kk * r * s * c
            nbytes += 2.0 * (n * h * w * c + kk * r * s * c + n * P * Q * kk)
        elif body["kind"] == "rmsnorm_bf16":
            nbytes += 2.0 * (2 * p[0] * p[1] + p[1])
        elif body["kind"] == "silu_mul_bf16":
            nbytes += 6.0 * p[0]
        elif body["kind"] == "attn_decode_bf16":
            nbytes += 2.0 * (2 * p[0] * 8 * 128 + 2 * 32 * 128)
        elif body["kind"] == "gemv_bf16":
            flops += 2.0 * p[0] * p[1]
            nbytes += 2.0 * (p[0] * p[1] + p[1] + p[0])
        else:
            nbytes += 8.0 * p[0] * k["blocks"]
    return {"kernels": len(kernels), "blocks": sum(k["blocks"] for k in kernels),
            "gflop": flops / 1e9, "gbytes": nbytes / 1e9}
