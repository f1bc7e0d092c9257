"""Two-layer expert predictors — the reference API over the B200 kernels.

Reference: pkg/src/moepredict/predictor.py. Names, signatures, shapes, the
1-D convenience form and the exception contract are kept:

    arch1: linear -> batch-norm -> GELU(tanh) -> dropout -> linear
    arch2: linear -> SiLU -> linear

`PredictorModel` stays a host object holding float64 parameters (so MOEPM1
checkpoints round-trip bit-exactly, predictor.py:354-412); every arithmetic
call uploads it into a `DevicePredictor` (engine.py) and runs the sm_100a
kernels. numpy in -> numpy float64 out; CUDA tensors in -> CUDA tensors out.
For a resident model across many calls use `DevicePredictor` directly.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from .core import ExpertSelection
from .engine import DevicePredictor
from .exceptions import BadMagicError, ConfigurationError, UsageError, VersionError

CHECKPOINT_MAGIC = b"MOEPM1"
CHECKPOINT_VERSION = 1
_CKPT_HEADER = struct.Struct("<5I")
ARCHS = ("arch1", "arch2")


@dataclass
class PredictorModel:
    """Parameters and normalisation state of one per-layer predictor
    (reference predictor.py:75-136)."""

    arch: str
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    bn_scale: np.ndarray | None = None
    bn_shift: np.ndarray | None = None
    bn_mean: np.ndarray | None = None
    bn_var: np.ndarray | None = None
    dropout_rate: float = 0.1
    bn_momentum: float = 0.1
    bn_eps: float = 1e-5
    mode: str = "eval"
    dropout_seed: int = 0
    _dropout_step: int = field(default=0, repr=False)
    _cache: dict | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.arch not in ARCHS:
            raise ConfigurationError(f"unknown arch {self.arch!r}")
        has_bn = all(v is not None for v in (self.bn_scale, self.bn_shift, self.bn_mean, self.bn_var))
        if self.arch == "arch1" and not has_bn:
            raise ConfigurationError("arch1 requires batch-norm state")
        if self.arch == "arch2" and has_bn:
            raise ConfigurationError("arch2 carries no batch-norm state")
        if self.bn_var is not None and np.any(np.asarray(self.bn_var) < 0):
            raise ConfigurationError("running variance must be >= 0")

    @property
    def d(self) -> int:
        return self.w1.shape[1]

    @property
    def hidden(self) -> int:
        return self.w1.shape[0]

    @property
    def n_experts(self) -> int:
        return self.w2.shape[0]

    def train(self) -> "PredictorModel":
        self.mode = "train"
        return self

    def eval(self) -> "PredictorModel":
        self.mode = "eval"
        self._cache = None
        return self

    def param_dict(self) -> dict:
        params = {"w1": self.w1, "b1": self.b1, "w2": self.w2, "b2": self.b2}
        if self.arch == "arch1":
            params["bn_scale"] = self.bn_scale
            params["bn_shift"] = self.bn_shift
        return params

    def to_device(self, device="cuda", **kw) -> DevicePredictor:
        return DevicePredictor(self, device, **kw)


def init_model(arch: str, d: int, hidden: int, n_experts: int, seed: int = 0,
               dropout_rate: float = 0.1) -> PredictorModel:
    """Kaiming-uniform fan-in init from the Philox(seed << 64) stream, so the
    parameters are bit-identical to the reference's (predictor.py:139-173)."""
    if arch not in ARCHS:
        raise ConfigurationError(f"unknown arch {arch!r}")
    rng = np.random.Generator(np.random.Philox(key=(int(seed) << 64)))
    w1 = rng.uniform(-np.sqrt(1.0 / d), np.sqrt(1.0 / d), size=(hidden, d))
    w2 = rng.uniform(-np.sqrt(1.0 / hidden), np.sqrt(1.0 / hidden), size=(n_experts, hidden))
    b1, b2 = np.zeros(hidden), np.zeros(n_experts)
    if arch == "arch1":
        return PredictorModel(arch, w1, b1, w2, b2, bn_scale=np.ones(hidden), bn_shift=np.zeros(hidden),
                              bn_mean=np.zeros(hidden), bn_var=np.ones(hidden),
                              dropout_rate=dropout_rate, dropout_seed=seed)
    return PredictorModel(arch, w1, b1, w2, b2, dropout_rate=0.0, dropout_seed=seed)


def n_params(model: PredictorModel) -> int:
    return int(sum(np.asarray(p).size for p in model.param_dict().values()))


def _as_batch(model: PredictorModel, x):
    """Shape contract of _check_input (predictor.py:180-190); finiteness is
    checked on the device by K0 and raised as ConfigurationError."""
    if isinstance(x, torch.Tensor):
        single = x.dim() == 1
        batch = x[None, :] if single else x
        if batch.dim() != 2 or batch.shape[1] != model.d:
            raise ConfigurationError(f"input shape {tuple(x.shape)} incompatible with d={model.d}")
        return batch, single, True
    x = np.asarray(x, dtype=np.float64)
    single = x.ndim == 1
    batch = x[None, :] if single else x
    if batch.ndim != 2 or batch.shape[1] != model.d:
        raise ConfigurationError(f"input shape {x.shape} incompatible with d={model.d}")
    return torch.from_numpy(np.ascontiguousarray(batch)), single, False


_DEV_CACHE: "dict[int, tuple]" = {}
_DEV_CACHE_MAX = 8
_SAMPLE = 4096


def _fingerprint(model) -> tuple:
    """Identity, buffer address, shape and a strided 4096-element sample of
    every parameter / BN array: an in-place update of the weights (the
    reference's optimizer, trainer.py:91-122, rewrites every element) or a new
    array changes it; a forced refresh is `device_for(model, refresh=True)`."""
    fp = [model.arch]
    for name in ("w1", "b1", "w2", "b2", "bn_scale", "bn_shift", "bn_mean", "bn_var"):
        a = getattr(model, name, None)
        if a is None:
            fp.append(None)
            continue
        a = np.asarray(a)
        flat = a.reshape(-1)
        step = max(1, flat.size // _SAMPLE)
        fp.append((id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str,
                   flat[::step][:_SAMPLE].tobytes(), flat[-1:].tobytes()))
    return tuple(fp)


def device_for(model, refresh: bool = False) -> DevicePredictor:
    """The HBM-resident DevicePredictor of a host model, uploaded once and
    reused while the model's parameters are unchanged (the reference API
    functions take host models; re-uploading 33.5 MB of fp64 W1 per call cost
    ~8x a 4k-token predict). Keyed by id(model) + _fingerprint; a small LRU."""
    key = id(model)
    fp = _fingerprint(model)
    hit = _DEV_CACHE.get(key)
    if hit is not None and not refresh and hit[0] == fp and hit[2]() is model:
        _DEV_CACHE[key] = _DEV_CACHE.pop(key)  # most recent last
        return hit[1]
    import weakref
    dev = DevicePredictor(model)
    try:
        ref = weakref.ref(model)
    except TypeError:  # an object without weakref support: keep it alive with the entry
        ref = (lambda m: (lambda: m))(model)
    _DEV_CACHE.pop(key, None)
    _DEV_CACHE[key] = (fp, dev, ref)
    while len(_DEV_CACHE) > _DEV_CACHE_MAX:
        _DEV_CACHE.pop(next(iter(_DEV_CACHE)))
    return dev


def predict_logits(model: PredictorModel, x):
    """Eval-mode logits regardless of the mode flag (predictor.py:330-334)."""
    batch, single, is_t = _as_batch(model, x)
    z = device_for(model).logits(batch.to("cuda"))
    if not is_t:
        z = z.cpu().numpy()
    return z[0] if single else z


def predict_topk_batch(model: PredictorModel, x, m: int):
    """Row-wise ascending top-m expert ids, shape (n, m) (predictor.py:347-351)."""
    if not 1 <= m <= model.n_experts:
        raise ValueError(f"m={m} out of range for {model.n_experts} experts")
    batch, single, is_t = _as_batch(model, x)
    dev = device_for(model)
    if not is_t:
        # numpy input: cast + predict without a host round trip in between; the
        # status decides after the (unavoidable) read of the ids
        spec = dev.topk_speculative(batch.to("cuda"), m)
        if spec is not None:
            ids, cst, kst = spec
            ids_np = ids.cpu().numpy().astype(np.int64)
            st = cst.cpu().numpy()
            if st[0]:
                raise ConfigurationError("input must be finite")
            if st[1] == 0:
                DevicePredictor.check_status(kst, batch)
                return ids_np
    ids = dev.topk(batch.to("cuda"), m).to(torch.int64)
    return ids if is_t else ids.cpu().numpy()


def predict_topk(model: PredictorModel, x, m: int) -> ExpertSelection:
    """Top-m selection for one activation vector (predictor.py:337-344)."""
    if model.mode != "eval":
        raise UsageError("predict_topk requires the model in eval mode")
    if not 1 <= m <= model.n_experts:
        raise ValueError(f"m={m} out of range for {model.n_experts} experts")
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    dev = device_for(model)
    batch = torch.from_numpy(x[None, :]).to("cuda")
    logits = dev.logits(batch)[0].cpu().numpy()
    ids = dev.topk(batch, m)[0].cpu().numpy()
    return ExpertSelection(indices=ids.astype(np.int64), raw_scores=logits)


def _trainer_fp64(model):
    from .losses import LossSpec
    from .train_engine import DeviceTrainer
    return DeviceTrainer(model, LossSpec(), precision="fp64")


def forward(model: PredictorModel, x, *, dropout_mask=None):
    """Predictor logits (predictor.py:243-258). Eval mode == predict_logits; train
    mode runs the fp64 device forward (K2 with pre-activation output; arch1 adds
    batch statistics, the running-stat update and the Philox dropout stream) and
    keeps the intermediates for a paired backward()."""
    if model.mode != "train":
        return predict_logits(model, x)
    batch, single, is_t = _as_batch(model, x)
    tr = _trainer_fp64(model)
    z, cache, xd = tr.forward(batch.to("cuda"), dropout_mask=dropout_mask, training=True)
    if model.arch == "arch1":
        # the reference mutates the running statistics and the dropout counter in place
        model.bn_mean[...] = tr.run_mean.cpu().numpy()
        model.bn_var[...] = tr.run_var.cpu().numpy()
        model._dropout_step = tr.dropout_step
    host_x = batch.detach().cpu().numpy().astype(np.float64) if is_t else batch.numpy()
    model._cache = {"x": host_x, "cache": cache, "x_dev": xd, "trainer": tr}
    out = z if is_t else z.cpu().numpy()
    return out[0] if single else out


def backward(model: PredictorModel, x, dlogits) -> dict:
    """Parameter gradients from upstream d(loss)/d(logits) (predictor.py:300-327),
    fp64 on the device: K5 for the activation / W2 / bias terms, an fp64 GEMM for dW1."""
    batch, single, is_t = _as_batch(model, x)
    dz = dlogits if isinstance(dlogits, torch.Tensor) else torch.as_tensor(np.asarray(dlogits, dtype=np.float64))
    dz = dz.to("cuda", torch.float64)
    if single:
        dz = dz[None]
    if tuple(dz.shape) != (batch.shape[0], model.n_experts):
        raise ConfigurationError(f"upstream gradient shape {tuple(dz.shape)} mismatches logits")
    if model.mode == "train":
        c = model._cache
        host_x = batch.detach().cpu().numpy().astype(np.float64) if is_t else batch.numpy()
        if c is None or c["x"].shape != host_x.shape or not np.array_equal(c["x"], host_x):
            raise UsageError("train-mode backward requires a paired forward on the same input")
        tr, cache, xd = c["trainer"], c["cache"], c["x_dev"]
    else:
        tr = _trainer_fp64(model)
        _, cache, xd = tr.forward(batch.to("cuda"), training=False)
    tr.backward(xd, cache, dz.contiguous())
    names = ("w1", "w2", "b1", "b2", "bn_scale", "bn_shift")[: len(tr.sizes)]
    return {n: tr.view(tr.grad, i).clone().cpu().numpy() for i, n in enumerate(names)}


def save_model(model: PredictorModel, path) -> None:
    """MOEPM1 checkpoint, float64 parameters in fixed order (predictor.py:354-369)."""
    arrays = [model.w1, model.b1, model.w2, model.b2]
    if model.arch == "arch1":
        arrays += [model.bn_scale, model.bn_shift, model.bn_mean, model.bn_var]
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(_CKPT_HEADER.pack(CHECKPOINT_VERSION, 1 if model.arch == "arch1" else 2,
                                  model.d, model.hidden, model.n_experts))
        f.write(struct.pack("<d", float(model.dropout_rate)))
        for arr in arrays:
            f.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def load_model(path) -> PredictorModel:
    """Read a MOEPM1 checkpoint; the model loads in eval mode (predictor.py:372-412)."""
    with open(path, "rb") as f:
        blob = f.read()
    if blob[: len(CHECKPOINT_MAGIC)] != CHECKPOINT_MAGIC:
        raise BadMagicError("not a predictor checkpoint")
    off = len(CHECKPOINT_MAGIC)
    version, arch_tag, d, hidden, e = _CKPT_HEADER.unpack_from(blob, off)
    off += _CKPT_HEADER.size
    if version != CHECKPOINT_VERSION:
        raise VersionError(f"unsupported checkpoint version {version}")
    if arch_tag not in (1, 2):
        raise ConfigurationError(f"unknown arch tag {arch_tag}")
    (dropout_rate,) = struct.unpack_from("<d", blob, off)
    off += 8

    def take(shape):
        nonlocal off
        count = int(np.prod(shape))
        arr = np.frombuffer(blob, dtype="<f8", count=count, offset=off)
        off += count * 8
        return arr.astype(np.float64).reshape(shape)

    w1, b1, w2, b2 = take((hidden, d)), take((hidden,)), take((e, hidden)), take((e,))
    if arch_tag == 1:
        return PredictorModel("arch1", w1, b1, w2, b2, bn_scale=take((hidden,)), bn_shift=take((hidden,)),
                              bn_mean=take((hidden,)), bn_var=take((hidden,)), dropout_rate=dropout_rate)
    return PredictorModel("arch2", w1, b1, w2, b2, dropout_rate=dropout_rate)
