"""K0 input norm (moep_input_norm) against the oracle's input_norm_bf16
(numpy fp64: core.layer_norm order, then bf16 RNE): bit-identical x_hat for
both kernels (the one-pass bf16 fast path for d in {512, 1024, 2048, 4096},
the general numpy-tree path otherwise), every norm kind, affine or not, and
rows built to stress the statistics (constant rows, huge / tiny values).
The fast path's rounding decision (reciprocal multiply unless the value is
near a bf16 midpoint) is checked against the forced exact chain on 2^30
elements."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_10676_b200.engine import input_norm
    return input_norm


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    return oracle


def _rows(rng, O, n, d):
    x = 3.0 * rng.standard_normal((n, d)) + 0.5
    x[0] = 1.25                               # constant row: var 0, sigma = sqrt(eps)
    x[1] = 0.0                                # zero row
    x[2, ::7] *= 1e4                          # wide range within a row
    x[3] *= 1e-30                             # tiny row (var far below eps)
    x[4, :] = rng.standard_normal(d) * 1e3    # large row
    return O.round_bf16(x)


CASES = [("rmsnorm", True, False), ("rmsnorm", False, False), ("layernorm", True, True),
         ("layernorm", False, False), ("layernorm", True, False)]


@pytest.mark.parametrize("d", [512, 1024, 2048, 4096, 1000, 136])
@pytest.mark.parametrize("xdt", ["bf16", "f64"])
def test_norm_bit_identical_to_oracle(K, O, d, xdt):
    rng = np.random.default_rng(d)
    n = 1031  # ragged row groups
    x = _rows(rng, O, n, d)
    xt = torch.from_numpy(x).cuda()
    xt = xt.to(torch.bfloat16) if xdt == "bf16" else xt
    gamma = rng.uniform(0.5, 1.5, d)
    beta = 0.1 * rng.standard_normal(d)
    for kind, g, b in CASES:
        out = K(xt, kind, gamma if g else None, beta if b else None).double().cpu().numpy()
        ref = O.input_norm_bf16(x, kind, gamma if g else None, beta if b else None)
        assert np.array_equal(out, ref), (kind, g, b)


@pytest.mark.parametrize("d", [2048, 4096])
def test_fast_path_rounding_decision_at_scale(K, O, d):
    """2^30 elements: the fast kernel (reciprocal multiply + midpoint test)
    equals the forced exact chain everywhere, and the oracle on a sample."""
    n = (1 << 30) // d
    g = torch.Generator(device="cuda")
    g.manual_seed(d)
    x = (torch.randn((n, d), device="cuda", generator=g) * 2.0 + 0.3).to(torch.bfloat16)
    rng = np.random.default_rng(1)
    gamma = rng.uniform(0.5, 1.5, d)
    beta = 0.1 * rng.standard_normal(d)
    for kind, b in (("rmsnorm", None), ("layernorm", beta)):
        fast = K(x, kind, gamma, b)
        exact = K(x, kind, gamma, b, _force_exact=True)
        assert torch.equal(fast, exact), kind
        rows = np.arange(0, n, n // 64)
        ref = O.input_norm_bf16(x[rows].double().cpu().numpy(), kind, gamma, b)
        assert np.array_equal(fast[rows].double().cpu().numpy(), ref), kind


def test_norm_nonfinite_and_shapes(K, O):
    from paper_2511_10676_b200.exceptions import ConfigurationError
    x = torch.zeros((64, 2048), dtype=torch.bfloat16, device="cuda")
    x[7, 3] = float("nan")
    with pytest.raises(ConfigurationError):
        K(x, "rmsnorm")
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    K(x, "layernorm", status=st)
    assert int(st[0]) == 1
    with pytest.raises(ConfigurationError):
        K(x[0], "rmsnorm")
    with pytest.raises(ConfigurationError):
        K(x, "batchnorm")
    # cast (kind none): exactness flag
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    xd = torch.full((4, 16), 1.0 + 2.0 ** -20, dtype=torch.float64, device="cuda")
    out = K(xd, "none", status=st)
    assert int(st[1]) > 0 and torch.equal(out.double(), torch.full_like(xd, 1.0))
