"""Pins of the oracle's NAG update (reading
R24): SPEC's hand-evaluated two steps, mu = 0 as plain SGD, the zero-gradient
case, and torch.optim.SGD(nesterov=True) (a library routine) with weight decay."""
import numpy as np
import torch

import oracle


def f32(*a):
    return [np.ascontiguousarray(x, dtype=np.float32) for x in a]


def test_spec_two_steps():
    # d=1, mu=0.9, eta=1, g~=1 twice: v=1, x1 = x0 - 1.9; v=1.9, x2 = x1 - 2.71
    g, vel, x = f32([1.0], [0.0], [5.0])
    oracle.nag(g, vel, x, 1.0, 0.9, 0.0)
    assert vel[0] == np.float32(1.0) and abs(x[0] - (5.0 - 1.9)) < 1e-6
    x1 = float(x[0])
    oracle.nag(g, vel, x, 1.0, 0.9, 0.0)
    assert abs(vel[0] - 1.9) < 1e-6 and abs(x[0] - (x1 - 2.71)) < 1e-6


def test_mu_zero_is_sgd():
    rng = np.random.default_rng(1)
    g, x0 = f32(rng.standard_normal(100), rng.standard_normal(100))
    vel, x = f32(np.zeros(100), x0.copy())
    oracle.nag(g, vel, x, 0.1, 0.0, 0.0)
    assert x.tobytes() == (x0 - np.float32(0.1) * g).tobytes()


def test_zero_gradient_zero_velocity_is_fixed_point():
    x0 = np.linspace(-1, 1, 33).astype(np.float32)
    g, vel, x = f32(np.zeros(33), np.zeros(33), x0.copy())
    oracle.nag(g, vel, x, 0.5, 0.9, 0.0)
    assert x.tobytes() == x0.tobytes()


def test_torch_sgd_nesterov_weight_decay():
    rng = np.random.default_rng(2)
    n, mu, lr, wd = 257, 0.9, 0.05, 0.01
    x0 = rng.standard_normal(n).astype(np.float32)
    p = torch.nn.Parameter(torch.tensor(x0, dtype=torch.float64))
    opt = torch.optim.SGD([p], lr=lr, momentum=mu, nesterov=True, weight_decay=wd)
    vel, x = f32(np.zeros(n), x0.copy())
    for _ in range(10):
        g = rng.standard_normal(n).astype(np.float32)
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        oracle.nag(g, vel, x, lr, mu, wd)
    np.testing.assert_allclose(x, p.detach().numpy(), rtol=1e-5, atol=1e-6)
