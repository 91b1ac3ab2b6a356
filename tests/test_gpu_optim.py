"""Adam on the device: svr_adam_step against the
unmodified reference adam_step (optim.cpp:322-345), bit for bit on the
float parameters and the fp64 moments, over several steps with the
reference's two learning-rate rules (uniform for densities; SH band 0 vs
the rest, optim.cpp:489-491)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("period,n_primary", [(0, 0), (48, 3)])
def test_adam_steps_bit_exact(svr, ctx, ref, period, n_primary):
    import torch
    rng = np.random.default_rng(11)
    n = 48 * 2000 + 7
    p0 = rng.normal(0, 1, n).astype(np.float32)
    dev = torch.device("cuda", 0)
    params = torch.tensor(p0, device=dev)
    st = svr.AdamState(n)
    p_ref, m_ref, v_ref = p0.copy(), np.zeros(n), np.zeros(n)
    for step in range(5):
        g = (rng.normal(0, 1e-2, n) * (rng.uniform(size=n) < 0.7)).astype(np.float32)
        svr.adam_step(ctx, params, torch.tensor(g, device=dev), st, 0.025, 0.00025, period,
                      n_primary)
        p_ref, m_ref, v_ref = ref.ref_adam_step(p_ref, g.astype(np.float64), m_ref, v_ref, step,
                                                0.025, 0.00025, period, n_primary)
    ctx.synchronize()
    assert np.array_equal(params.cpu().numpy(), p_ref)
    assert np.array_equal(st.m.cpu().numpy(), m_ref)
    assert np.array_equal(st.v.cpu().numpy(), v_ref)


def test_adam_nan_gradient_raises(svr, ctx):
    import torch
    dev = torch.device("cuda", 0)
    params = torch.zeros(100, device=dev)
    g = torch.zeros(100, device=dev)
    g[37] = float("nan")
    with pytest.raises(RuntimeError):
        svr.adam_step(ctx, params, g, svr.AdamState(100), 0.01)


def test_adam_deferred_nan_check(svr, ctx):
    """Deferred Adam (on_device = 2) returns at once; a NaN gradient is
    reported (and cleared) by svr_ctx_take_adam_nan."""
    import ctypes as C
    import torch
    dev = torch.device("cuda", 0)
    lib = ctx._lib
    params = torch.zeros(100, device=dev)
    m = torch.zeros(100, dtype=torch.float64, device=dev)
    v = torch.zeros(100, dtype=torch.float64, device=dev)
    g = torch.zeros(100, device=dev)
    torch.cuda.synchronize()
    nan = C.c_int32()

    def step(grad):
        svr._check(lib.svr_adam_step(ctx.h, C.c_void_p(params.data_ptr()), C.c_void_p(grad.data_ptr()),
                                     C.c_void_p(m.data_ptr()), C.c_void_p(v.data_ptr()), 100, 1, 0.01,
                                     0.0, 0, 0, 0.1, 0.99, 1e-15, 2))

    step(g)
    svr._check(lib.svr_ctx_take_adam_nan(ctx.h, C.byref(nan)))
    assert nan.value == 0
    g[37] = float("nan")
    torch.cuda.synchronize()
    step(g)
    svr._check(lib.svr_ctx_take_adam_nan(ctx.h, C.byref(nan)))
    assert nan.value == 1
    svr._check(lib.svr_ctx_take_adam_nan(ctx.h, C.byref(nan)))
    assert nan.value == 0
