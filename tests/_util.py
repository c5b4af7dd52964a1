"""Shared test helpers: move device tensors to the oracle's storage form and apply the tolerances.

Tolerances (BASELINE.json north_star):
  * search: idx/hit bit-exact where the oracle's top-1/top-2 gap (idx) or |s1 - tau| (hit)
    exceeds 1e-4 (reading R5); otherwise the GPU's pick must score within 1e-4 of the best.
    |score_gpu - s_oracle(idx_gpu)| <= 5e-5: half the 1e-4 decision margin, so two scores more
    than 1e-4 apart can never swap order (tcgen05 fp32 accumulation
    measured 1.1e-5 max at D=4096, the a-priori bound D*2^-24 is 2.4e-4).
  * bf16/fp16 outputs: max-abs <= 2e-2 over all elements and rel-L2 <= 5e-3 per unit.
  * fp32 outputs (tiny config, CUDA-core fp32 accumulation over <= 32 terms): max-abs <= 1e-4,
    rel-L2 <= 1e-5 per unit.
"""
import numpy as np
import torch

import oracle

DT_NAME = {torch.float32: "f32", torch.float16: "f16", torch.bfloat16: "bf16"}


def storage(t: torch.Tensor) -> np.ndarray:
    """Exact bytes of a tensor as the oracle's numpy storage (bf16 -> uint16 bit patterns)."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def check_search(q, x, idx, score, hit, tau, gbase=0):
    """A5 exactness rule against the brute-force oracle (x is the full DB: global indices)."""
    dt = DT_NAME[q.dtype]
    qs, xs = storage(q), storage(x)
    i_o, s1, s2, h_o = oracle.search(qs, xs, dt, tau)
    idx, score, hit = idx.cpu().numpy(), score.cpu().numpy().astype(np.float64), hit.cpu().numpy()
    B = len(idx)
    assert np.all((idx >= 0) & (idx < xs.shape[0])), "index out of range"
    strict = (s1 - s2) > 1e-4
    bad = np.nonzero(strict & (idx != i_o))[0]
    assert bad.size == 0, f"idx differs at {bad[:10]}: gpu {idx[bad[:10]]} oracle {i_o[bad[:10]]}"
    s_at = oracle.scores(qs, xs, dt, np.arange(B), idx)
    assert np.all(s_at >= s1 - 1e-4), "GPU pick is not a near-best entry"
    assert np.max(np.abs(score - s_at), initial=0) <= 5e-5, f"score error {np.max(np.abs(score - s_at))}"
    far = np.abs(s1 - np.float64(np.float32(tau))) > 1e-4
    bad = np.nonzero(far & (hit != h_o))[0]
    assert bad.size == 0, f"hit differs at {bad[:10]}"
    assert np.array_equal(hit.astype(bool), score >= np.float32(tau)), "hit != (score >= tau)"
    return i_o, s1, s2, h_o


def tolerances(dtype):
    if dtype == torch.float32:
        return 1e-4, 1e-5
    return 2e-2, 5e-3


def check_close(got: torch.Tensor, ref: np.ndarray, dtype, what=""):
    """got: device/host tensor [U][S][d] (any float dtype), ref: f64 [U][S][d]."""
    g = got.detach().double().cpu().numpy().reshape(ref.shape)
    max_abs_tol, rel_tol = tolerances(dtype)
    err = np.abs(g - ref)
    assert np.all(np.isfinite(g)), f"{what}: non-finite output"
    ma = float(err.max(initial=0))
    assert ma <= max_abs_tol, f"{what}: max-abs {ma} > {max_abs_tol}"
    num = np.sqrt((err.reshape(len(ref), -1) ** 2).sum(1))
    den = np.sqrt((ref.reshape(len(ref), -1) ** 2).sum(1))
    rel = num / np.maximum(den, 1e-30)
    assert rel.max(initial=0) <= rel_tol, f"{what}: rel-L2 {rel.max()} > {rel_tol}"
    return ma, float(rel.max(initial=0))
