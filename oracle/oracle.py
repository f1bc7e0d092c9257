"""CPU oracle for the B200 expert-predictor path — TEST INFRASTRUCTURE ONLY.

This module restates, in float64 numpy, the reference algorithm of
arXiv 2511.10676's `moepredict` package for the hot path (predictor forward /
selection, evaluation reductions, losses, backward, optimizer step). It is the
checker the parity tests compare the CUDA path against, and the CPU baseline
`bench.py` times. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu-baseline / reference arm may import it; the product package
(`paper_2511_10676_b200`) never does.

Pinning: `tests/test_oracle_golden.py` checks every function here against
(a) the known-answer values in the reference's own tests and (b) golden
fixtures produced by importing the real reference in the build container
(`tests/golden/make_golden.py` → `tests/golden/*.npz`).

Citations `core.py:NN` etc. refer to /root/reference/pkg/src/moepredict/.
"""

from __future__ import annotations

import numpy as np

TOP_TIER_SIZE = 10  # losses.py:27
MID_TIER_SIZE = 30  # losses.py:28
LAYER_NORM_EPS = 1e-5  # core.py:16
GELU_C = np.sqrt(2.0 / np.pi)  # predictor.py:35
GELU_A = 0.044715  # predictor.py:36


# --------------------------------------------------------------------- core
def softmax(z, axis=-1):
    """Max-subtracted softmax (core.py:19-24)."""
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max(axis=axis, keepdims=True))
    return e / e.sum(axis=axis, keepdims=True)


def rank_order(scores):
    """Descending order, ties to the lower index: stable argsort of -s (core.py:51-54)."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    return np.argsort(-s, axis=1, kind="stable")


def top_k_batch(scores, k):
    """First k of the stable descending order, returned ascending (core.py:42-48)."""
    s = np.asarray(scores, dtype=np.float64)
    if not 1 <= k <= s.shape[1]:
        raise ValueError(f"k={k} out of range for {s.shape[1]} scores")
    return np.sort(rank_order(s)[:, :k], axis=1)


def top_k(scores, k):
    """1-D form of top_k_batch (core.py:27-39)."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise ValueError("scores must be 1-D")
    return top_k_batch(s[None, :], k)[0]


def layer_norm(x, eps=LAYER_NORM_EPS):
    """Non-affine layer norm, population variance (core.py:57-68)."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


# ------------------------------------------------------ bf16 + input norm
def round_bf16(x):
    """float64 -> nearest bf16 value (round-half-even), returned as float64.

    Direct fp64->bf16 rounding (no fp32 double rounding); values beyond the
    bf16 range become +-inf, values below the bf16 subnormal quantum use the
    fixed 2^-133 quantum.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    fin = np.isfinite(x)
    out[~fin] = x[~fin]
    xf = x[fin]
    m, e = np.frexp(xf)  # xf = m * 2^e, 0.5 <= |m| < 1
    normal = e >= -125  # |x| >= 2^-126
    r = np.empty_like(xf)
    r[normal] = np.ldexp(np.rint(m[normal] * 256.0), e[normal] - 8)
    q = 2.0 ** -133
    r[~normal] = np.rint(xf[~normal] / q) * q
    r[np.abs(r) > 3.3895313892515355e38] = np.inf * np.sign(r[np.abs(r) > 3.3895313892515355e38])
    out[fin] = r
    return out


def input_norm_bf16(x, kind="none", gamma=None, beta=None, eps=None):
    """Pre-attention input norm feeding the predictor, rounded to bf16.

    The reference predictor consumes the model's `input_layernorm` output
    (exporter hooks.py:19,113-114); its only norm is core.layer_norm. The B200
    path fuses the real models' norms: rmsnorm (DeepSeek-V2 / Qwen3-MoE,
    eps 1e-6) and affine layernorm (Phi-MoE, eps 1e-5) — statistics in fp64,
    output rounded fp64 -> bf16 RNE.
    """
    x = np.asarray(x, dtype=np.float64)
    if kind == "none":
        return round_bf16(x)
    if kind == "rmsnorm":
        eps = 1e-6 if eps is None else eps
        ms = np.mean(x * x, axis=-1, keepdims=True)
        y = x / np.sqrt(ms + eps)
        if gamma is not None:
            y = y * np.asarray(gamma, dtype=np.float64)
        return round_bf16(y)
    if kind == "layernorm":
        eps = LAYER_NORM_EPS if eps is None else eps
        y = layer_norm(x, eps)
        if gamma is not None:
            y = y * np.asarray(gamma, dtype=np.float64)
        if beta is not None:
            y = y + np.asarray(beta, dtype=np.float64)
        return round_bf16(y)
    raise ValueError(f"unknown norm kind {kind!r}")


# ------------------------------------------------------------- predictor
def sigmoid(u):
    """Branch-stable logistic (predictor.py:39-45; losses.py:134-140)."""
    u = np.asarray(u, dtype=np.float64)
    out = np.empty_like(u)
    pos = u >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-u[pos]))
    eu = np.exp(u[~pos])
    out[~pos] = eu / (1.0 + eu)
    return out


def silu(u):
    return u * sigmoid(u)  # predictor.py:48-49


def silu_grad(u):
    s = sigmoid(u)  # predictor.py:52-54
    return s * (1.0 + u * (1.0 - s))


def gelu_tanh(u):
    t = np.tanh(GELU_C * (u + GELU_A * u**3))  # predictor.py:57-61
    return 0.5 * u * (1.0 + t)


def gelu_tanh_grad(u):
    t = np.tanh(GELU_C * (u + GELU_A * u**3))  # predictor.py:64-67
    dt = (1.0 - t**2) * GELU_C * (1.0 + 3.0 * GELU_A * u**2)
    return 0.5 * (1.0 + t) + 0.5 * u * dt


def init_params(arch, d, hidden, n_experts, seed=0):
    """Kaiming-uniform fan-in init from a Philox(seed << 64) stream (predictor.py:139-173).

    Returns a dict with w1, b1, w2, b2 (+ bn_scale/shift/mean/var for arch1).
    """
    rng = np.random.Generator(np.random.Philox(key=(int(seed) << 64)))
    lim1, lim2 = np.sqrt(1.0 / d), np.sqrt(1.0 / hidden)
    p = {
        "arch": arch,
        "w1": rng.uniform(-lim1, lim1, size=(hidden, d)),
        "w2": rng.uniform(-lim2, lim2, size=(n_experts, hidden)),
        "b1": np.zeros(hidden),
        "b2": np.zeros(n_experts),
    }
    if arch == "arch1":
        p.update(bn_scale=np.ones(hidden), bn_shift=np.zeros(hidden),
                 bn_mean=np.zeros(hidden), bn_var=np.ones(hidden), bn_eps=1e-5)
    return p


def forward_eval(p, x):
    """Eval-mode logits and the cache backward needs (predictor.py:193-240, training=False)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    a = x @ p["w1"].T + p["b1"]
    cache = {"x": x, "a": a}
    if p["arch"] == "arch2":
        h = silu(a)
    else:
        inv_std = 1.0 / np.sqrt(p["bn_var"] + p.get("bn_eps", 1e-5))
        a_hat = (a - p["bn_mean"]) * inv_std
        bn_out = p["bn_scale"] * a_hat + p["bn_shift"]
        h = gelu_tanh(bn_out)
        cache.update(a_hat=a_hat, inv_std=inv_std, bn_out=bn_out)
    cache["h"] = h
    return h @ p["w2"].T + p["b2"], cache


def predict_logits(p, x):
    return forward_eval(p, x)[0]  # predictor.py:330-334


def predict_topk_batch(p, x, m):
    return top_k_batch(predict_logits(p, x), m)  # predictor.py:347-351


def backward_eval(p, cache, dz):
    """Parameter gradients from the eval cache (predictor.py:261-297, training=False)."""
    dz = np.atleast_2d(np.asarray(dz, dtype=np.float64))
    g = {"w2": dz.T @ cache["h"], "b2": dz.sum(axis=0)}
    dh = dz @ p["w2"]
    if p["arch"] == "arch2":
        da = dh * silu_grad(cache["a"])
    else:
        dbn = dh * gelu_tanh_grad(cache["bn_out"])
        g["bn_scale"] = (dbn * cache["a_hat"]).sum(axis=0)
        g["bn_shift"] = dbn.sum(axis=0)
        da = dbn * p["bn_scale"] * cache["inv_std"]
    g["w1"] = da.T @ cache["x"]
    g["b1"] = da.sum(axis=0)
    return g


# ------------------------------------------------------------------ losses
def batch_labels(scores, k):
    """topk_mask and 1-based stable rank (losses.py:64-74)."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    n, e = s.shape
    mask = np.zeros((n, e), dtype=bool)
    mask[np.arange(n)[:, None], top_k_batch(s, k)] = True
    ranks = np.empty((n, e), dtype=np.int64)
    ranks[np.arange(n)[:, None], rank_order(s)] = np.arange(1, e + 1)
    return {"true_scores": s, "topk_mask": mask, "rank_of": ranks}


def _softplus(z):
    return np.logaddexp(0.0, z)  # losses.py:86-87


def tier_weights(lab, top_w, rest_w, mid_w=None):
    """losses.py:113-121."""
    e = lab["rank_of"].shape[1]
    top_cut = min(TOP_TIER_SIZE, e)
    w = np.full(lab["rank_of"].shape, rest_w, dtype=np.float64)
    if mid_w is not None:
        mid_cut = min(MID_TIER_SIZE, e)
        w[(lab["rank_of"] > top_cut) & (lab["rank_of"] <= mid_cut)] = mid_w
    w[lab["rank_of"] <= top_cut] = top_w
    return w


def weighted_bce(z, lab, w):
    """losses.py:124-131."""
    n, e = z.shape
    t = lab["topk_mask"]
    logs = np.where(t, -_softplus(-z), -_softplus(z))
    return float(-np.sum(w * logs) / (n * e)), w * (sigmoid(z) - t) / (n * e)


def focal(z, lab, gamma=2.0, alpha=0.25):
    """losses.py:156-179."""
    n, e = z.shape
    pos = lab["topk_mask"]
    log_pt = np.where(pos, -_softplus(-z), -_softplus(z))
    pt = np.exp(log_pt)
    at = np.where(pos, alpha, 1.0 - alpha)
    loss = float(np.sum(-at * (1.0 - pt) ** gamma * log_pt) / (n * e))
    sgn = np.where(pos, 1.0, -1.0)
    d = at * sgn * (gamma * pt * (1.0 - pt) ** gamma * log_pt - (1.0 - pt) ** (gamma + 1.0))
    return loss, d / (n * e)


def mse_probs(probs, lab):
    """losses.py:99-110 (gradient w.r.t. probabilities)."""
    n = probs.shape[0]
    diff = lab["true_scores"] - probs
    return float(np.sum(diff * diff) / n), -2.0 * diff / n


def ranking_hinge(z, lab, margin=0.1, normalize=True):
    """Pairwise hinge over the true top-T, strict true-score pairs (losses.py:182-217).

    Vectorised restatement of the per-row loop: pair (j, l) counts when both
    are in the true top-T (rank <= T) and s_j > s_l strictly.
    """
    n, e = z.shape
    top_cut = min(TOP_TIER_SIZE, e)
    intop = lab["rank_of"] <= top_cut
    s = lab["true_scores"]
    higher = (s[:, :, None] > s[:, None, :]) & intop[:, :, None] & intop[:, None, :]
    n_pairs = int(higher.sum())
    gap = margin - (z[:, :, None] - z[:, None, :])
    viol = higher & (gap > 0)
    total = float(np.sum(np.where(viol, gap, 0.0)))
    grad = viol.sum(axis=1).astype(np.float64) - viol.sum(axis=2).astype(np.float64)
    if normalize and n_pairs > 0:
        total /= n_pairs
        grad /= n_pairs
    return total, grad, n_pairs


def loss_and_grad(spec, z, lab):
    """Dispatch over the four families (losses.py:243-273). `spec` is a dict."""
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    fam = spec.get("family", "wbce")
    if fam == "mse":
        probs = softmax(z, axis=1)
        loss, dp = mse_probs(probs, lab)
        inner = np.sum(dp * probs, axis=1, keepdims=True)
        return loss, probs * (dp - inner)
    if fam == "wbce":
        w = tier_weights(lab, spec.get("top_weight", 3.0), spec.get("rest_weight", 0.5))
        return weighted_bce(z, lab, w)
    if fam == "focal":
        return focal(z, lab, spec.get("focal_gamma", 2.0), spec.get("focal_alpha", 0.25))
    w = tier_weights(lab, spec.get("top_weight", 3.0), spec.get("rest_weight", 0.5),
                     spec.get("mid_weight", 1.5))
    bce, gb = weighted_bce(z, lab, w)
    hinge, gh, _ = ranking_hinge(z, lab, spec.get("margin", 0.1), spec.get("normalize_ranking", True))
    lam = spec.get("ranking_lambda", 0.3)
    return bce + lam * hinge, gb + lam * gh


# ----------------------------------------------------------------- metrics
def default_m_list(k, e):
    return sorted({k, min(k + 4, e), e})  # metrics.py:133-135


def eval_counters(z, truth, e, m_list=None):
    """Integer counters behind evaluate_predictions (metrics.py:138-193).

    Returns a dict: n, m_values, overprov_count[m], recall_count[m], top1_count,
    per_expert_hits[E], per_expert_truth[E]; means are count / n (or / n*k).
    """
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    truth = np.atleast_2d(np.asarray(truth, dtype=np.int64))
    n, k = truth.shape
    ms = sorted(set(default_m_list(k, e) if m_list is None else m_list))
    if k not in ms:
        ms.insert(0, k)
    order = rank_order(z)
    rows = np.arange(n)[:, None]
    pred_rank = np.empty_like(order)
    pred_rank[rows, order] = np.arange(e)[None, :]
    tr = pred_rank[rows, truth]
    out = {"n": n, "k": k, "m_values": ms,
           "overprov_count": {m: int((tr < m).all(axis=1).sum()) for m in ms},
           "recall_count": {m: int((tr < m).sum()) for m in ms},
           "top1_count": int((tr == 0).any(axis=1).sum()),
           "per_expert_hits": np.bincount(truth[tr < k].ravel(), minlength=e).astype(np.int64),
           "per_expert_truth": np.bincount(truth.ravel(), minlength=e).astype(np.int64)}
    return out


def evaluate_predictions(z, truth, e, m_list=None):
    """Means exactly as metrics.py:165-193 computes them (float of a bool mean)."""
    c = eval_counters(z, truth, e, m_list)
    n, k = c["n"], c["k"]
    overprov = {m: float(np.float64(c["overprov_count"][m]) / n) for m in c["m_values"]}
    recall = {m: float(np.float64(c["recall_count"][m]) / (n * k)) for m in c["m_values"]}
    return {"exact_match": overprov[k], "top1": float(np.float64(c["top1_count"]) / n),
            "overprov": overprov, "overprov_recall": recall,
            "per_expert_hits": c["per_expert_hits"], "per_expert_truth": c["per_expert_truth"],
            "n_samples": n, "k": k}


def tier_profile(scores):
    """Mean of the r-th largest score (metrics.py:47-57)."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    return np.sort(s, axis=1)[:, ::-1].mean(axis=0)


# --------------------------------------------------------------- optimizer
def adam_step(params, grads, state, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """In-place Adam with bias correction (trainer.py:103-122). `t` is the 1-based step."""
    for name, g in grads.items():
        st = state.setdefault(name, {"m": np.zeros_like(g), "v": np.zeros_like(g)})
        st["m"] *= b1
        st["m"] += (1 - b1) * g
        st["v"] *= b2
        st["v"] += (1 - b2) * g * g
        m_hat = st["m"] / (1 - b1**t)
        v_hat = st["v"] / (1 - b2**t)
        params[name] -= lr * m_hat / (np.sqrt(v_hat) + eps)


def sgd_step(params, grads, state, lr, momentum=None):
    """trainer.py:109-114."""
    for name, g in grads.items():
        if momentum is None:
            params[name] -= lr * g
        else:
            st = state.setdefault(name, {"m": np.zeros_like(g)})
            st["m"] *= momentum
            st["m"] += g
            params[name] -= lr * st["m"]


# ------------------------------------------------------- synthetic inputs
def teacher_scores(x, gate_w):
    """Router ground truth for synthetic activations: softmax(W_g . layer_norm(x))
    (synthgen.py:185-188 with post_norm=True; core.py:117-127)."""
    return softmax(layer_norm(x) @ np.asarray(gate_w, dtype=np.float64).T, axis=-1)


# ------------------------------------------------------------ train loop
def train_arch2(acts, scores, topk, k, *, hidden=32, batch_size=64, epochs=1, lr=1e-3, optimizer="adam",
                seed=0, eval_fraction=0.1, loss=None, overprov_m=None, max_steps=None, arch="arch2"):
    """Restatement of trainer.train for arch2 (trainer.py:131-204): Philox
    shuffle/split, labels from the fp64 cast of the fp32 scores, minibatch
    forward / loss_and_grad / backward / optimizer, held-out eval per epoch.
    Returns (params, [(train_loss, exact, top1, overprov)], steps)."""
    loss = loss or {"family": "wbce"}
    n = acts.shape[0]
    d, e = acts.shape[1], scores.shape[1]
    m_over = overprov_m if overprov_m else min(e, k + 4)
    rng = np.random.Generator(np.random.Philox(key=((int(seed) & 0xFFFFFFFFFFFFFFFF) << 64) + (1 << 61) + 7))
    perm = rng.permutation(n)
    n_eval = max(1, int(round(n * eval_fraction)))
    tr_idx, ev_idx = perm[: n - n_eval], perm[n - n_eval:]
    x_tr = acts[tr_idx].astype(np.float64)
    lab = batch_labels(scores[tr_idx].astype(np.float64), k)
    x_ev, tk_ev = acts[ev_idx].astype(np.float64), topk[ev_idx]
    p = init_params(arch, d, hidden, e, seed=seed)
    drop = {"seed": seed, "step": 0}
    names = ("w1", "b1", "w2", "b2") + (("bn_scale", "bn_shift") if arch == "arch1" else ())
    state, t, steps, rows = {}, 0, 0, []
    for _ in range(epochs):
        order = rng.permutation(x_tr.shape[0])
        loss_sum = 0.0
        for start in range(0, x_tr.shape[0], batch_size):
            b = order[start: start + batch_size]
            lb = {kk: v[b] for kk, v in lab.items()}
            if arch == "arch1":
                z, cache = forward_train_arch1(p, x_tr[b], drop)
            else:
                z, cache = forward_eval(p, x_tr[b])  # arch2 train forward == eval forward
            lv, dz = loss_and_grad(loss, z, lb)
            if not np.isfinite(lv):  # trainer.py:184-185
                raise FloatingPointError(f"non-finite loss at step {steps}")
            g = backward_train_arch1(p, cache, dz) if arch == "arch1" else backward_eval(p, cache, dz)
            g = {kk: g[kk] for kk in names}
            t += 1
            if optimizer == "adam":
                adam_step(p, g, state, t, lr=lr)
            else:
                sgd_step(p, g, state, lr, momentum=0.9 if optimizer == "momentum" else None)
            for nm in names:  # _nan_guard, trainer.py:125-128
                if not np.all(np.isfinite(p[nm])):
                    raise FloatingPointError(f"non-finite {nm} after step {steps}")
            loss_sum += lv * len(b)
            steps += 1
            if max_steps and steps >= max_steps:
                return p, rows, steps
        res = evaluate_predictions(predict_logits(p, x_ev), tk_ev, e, [m_over])
        rows.append((loss_sum / x_tr.shape[0], res["exact_match"], res["top1"], res["overprov"][m_over]))
    return p, rows, steps


# ------------------------------------------------ arch1 train mode (BN + dropout)
def forward_train_arch1(p, x, state, dropout_mask=None, momentum=0.1, rate=0.1):
    """Train-mode arch1 forward (predictor.py:208-237): batch statistics, running
    update (unbiased variance), Philox(seed << 64 + step) dropout. `state` holds
    'seed' and 'step' (advanced when a mask is drawn). Mutates p's bn_mean/bn_var."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    a = x @ p["w1"].T + p["b1"]
    mu, var = a.mean(axis=0), a.var(axis=0)
    inv_std = 1.0 / np.sqrt(var + p.get("bn_eps", 1e-5))
    a_hat = (a - mu) * inv_std
    n = a.shape[0]
    var_run = var * (n / (n - 1)) if n > 1 else var
    p["bn_mean"] *= 1.0 - momentum
    p["bn_mean"] += momentum * mu
    p["bn_var"] *= 1.0 - momentum
    p["bn_var"] += momentum * var_run
    bn_out = p["bn_scale"] * a_hat + p["bn_shift"]
    g = gelu_tanh(bn_out)
    if rate > 0:
        if dropout_mask is None:
            key = ((int(state["seed"]) & 0xFFFFFFFFFFFFFFFF) << 64) + int(state["step"])
            dropout_mask = np.random.Generator(np.random.Philox(key=key)).random(g.shape) >= rate
            state["step"] += 1
        keep = dropout_mask.astype(np.float64) / (1.0 - rate)
        h = g * keep
    else:
        keep = None
        h = g
    cache = {"x": x, "a": a, "a_hat": a_hat, "inv_std": inv_std, "bn_out": bn_out, "keep": keep, "h": h}
    return h @ p["w2"].T + p["b2"], cache


def backward_train_arch1(p, cache, dz):
    """predictor.py:261-297 with training=True (batch-statistics backward)."""
    dz = np.atleast_2d(np.asarray(dz, dtype=np.float64))
    g = {"w2": dz.T @ cache["h"], "b2": dz.sum(axis=0)}
    dh = dz @ p["w2"]
    dg = dh * cache["keep"] if cache["keep"] is not None else dh
    dbn = dg * gelu_tanh_grad(cache["bn_out"])
    g["bn_scale"] = (dbn * cache["a_hat"]).sum(axis=0)
    g["bn_shift"] = dbn.sum(axis=0)
    da_hat = dbn * p["bn_scale"]
    n = cache["a"].shape[0]
    a_hat = cache["a_hat"]
    da = cache["inv_std"] / n * (n * da_hat - da_hat.sum(axis=0) - a_hat * (da_hat * a_hat).sum(axis=0))
    g["w1"] = da.T @ cache["x"]
    g["b1"] = da.sum(axis=0)
    return g
