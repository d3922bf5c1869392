"""Pins for oracle/noise.py (PAPER.md P99-109, P150; SURVEY §8c-N, §8c pin table "Noise O6").

* Philox4x32-10 block == cuRAND's curand_Philox4x32_10 (textbook routine, host build)
* ln_fixed / cos2pi_fixed agree with libm within a few ulp (a dropped series
  term or wrong quadrant shows up as >=1e-9 errors)
* z ~ N(0,1): moments + Kolmogorov-Smirnov; Cov(W) ~= M_L (SPEC S255, S532)
"""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import fem, noise
from oracle.mesh import build_mesh
from synth import single_edge, tadpole


@pytest.fixture(scope="module")
def curand_kat(tmp_path_factory, repo_root):
    if shutil.which("g++") is None or not os.path.exists("/usr/local/cuda/include/curand_philox4x32_x.h"):
        pytest.skip("g++ or cuRAND header unavailable")
    d = tmp_path_factory.mktemp("kat")
    exe = str(d / "kat")
    subprocess.check_call(["g++", "-O2", "-I/usr/local/cuda/include",
                           os.path.join(repo_root, "tests", "kat", "curand_philox_host.cpp"), "-o", exe])
    return exe


def test_philox_matches_curand(curand_kat):
    rng = np.random.default_rng(1234)
    words = rng.integers(0, 2 ** 32, size=(2000, 6), dtype=np.uint64)
    words[0] = 0
    words[1] = 2 ** 32 - 1
    inp = "\n".join(" ".join(str(int(w)) for w in row) for row in words) + "\n"
    out = subprocess.run([curand_kat], input=inp, capture_output=True, text=True, check=True).stdout
    ref = np.array([[int(t) for t in line.split()] for line in out.strip().splitlines()], dtype=np.uint64)
    got = np.stack(noise.philox4x32_10(*[words[:, i] for i in range(6)]), axis=1)
    assert np.array_equal(got, ref)


def test_uniform_ranges():
    x0 = np.array([0, 0xFFFFFFFF], dtype=np.uint64)
    x1 = np.array([0, 0xFFFFFFFF], dtype=np.uint64)
    u1, u2 = noise.uniforms(x0, x1, x0, x1)
    assert u1[0] == 2.0 ** -53 and u1[1] == 1.0
    assert u2[0] == 0.0 and u2[1] == 1.0 - 2.0 ** -53


def _ulp_err(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_ln_fixed_vs_libm():
    rng = np.random.default_rng(7)
    x = np.concatenate([(rng.integers(1, 2 ** 53, 200000) + 0.0) * 2.0 ** -53,
                        [2.0 ** -53, 0.5, SQ := math.sqrt(0.5), SQ * (1 + 2 ** -52), 1.0 - 2 ** -53, 1.0]])
    got = noise.ln_fixed(x)
    ref = np.array([math.log(v) for v in x])
    nz = ref != 0
    assert got[~nz].tolist() == [0.0]
    assert _ulp_err(got[nz], ref[nz]).max() <= 4.0


def test_cos2pi_fixed_vs_libm():
    rng = np.random.default_rng(8)
    u = np.concatenate([rng.integers(0, 2 ** 53, 200000) * 2.0 ** -53,
                        [0.0, 0.125, 0.25, 0.375, 0.5, 0.625, 0.75, 0.875, 1 - 2.0 ** -53]])
    got = noise.cos2pi_fixed(u)
    ref = np.array([math.cos(2 * math.pi * v) for v in u])
    # libm's own argument 2*pi*u is rounded (|err| <= 2 pi * 2^-53 ~ 7e-16)
    assert np.max(np.abs(got - ref)) < 1.5e-15
    assert got[-5] == -1.0 and got[-9] == 1.0  # u = 0.5, u = 0


def test_standard_normal_statistics():
    from scipy import stats
    z = noise.standard_normal(seed=0, sample=0, dofs=np.arange(1_000_000))
    n = len(z)
    assert abs(z.mean()) < 5 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # different samples are independent streams
    z1 = noise.standard_normal(seed=0, sample=1, dofs=np.arange(100_000))
    assert abs(np.corrcoef(z[:100_000], z1)[0, 1]) < 5 / math.sqrt(100_000)


def test_seed_offset_convention():
    """Sample j of base seed s uses key s+j: grf_sample(seed=s0, n=1) == sample s0 of seed 0."""
    ML = np.ones(64)
    a = noise.white_noise(ML, seed=0, n_samples=5)[3]
    b = noise.white_noise(ML, seed=3, n_samples=1)[0]
    assert np.array_equal(a, b)


def test_noise_covariance_is_lumped_mass():
    """Cov(W) = M_L within 5 standard errors over 2e5 draws (SPEC S255, S532)."""
    mesh = build_mesh(tadpole(), 0.25)  # N small
    ML = fem.lumped_mass(mesh)
    n = 200_000
    # samples j = 0..n-1 of base seed 0 (key = j), vectorised over (sample, DOF)
    dofs = np.arange(mesh.n_dofs, dtype=np.uint64)
    keys = np.arange(n, dtype=np.uint64)
    K = np.repeat(keys, len(dofs))
    D = np.tile(dofs, n)
    zero = np.zeros_like(D)
    x = noise.philox4x32_10(D & noise._MASK, D >> noise._S32, zero, zero, K & noise._MASK, K >> noise._S32)
    u1, u2 = noise.uniforms(*x)
    z = (np.sqrt(-2.0 * noise.ln_fixed(u1)) * noise.cos2pi_fixed(u2)).reshape(n, len(dofs))
    W = z * np.sqrt(ML)[None, :]
    C = W.T @ W / n
    se_diag = np.sqrt(2.0 / n) * ML
    assert np.all(np.abs(np.diag(C) - ML) < 5 * se_diag)
    off = C - np.diag(np.diag(C))
    se_off = np.sqrt(np.outer(ML, ML) / n)
    assert np.all(np.abs(off) < 5 * se_off + np.eye(len(ML)))


def test_white_noise_scaling():
    mesh = build_mesh(single_edge(1.0), 0.25)
    ML = fem.lumped_mass(mesh)
    W = noise.white_noise(ML, 5, 2)
    z = np.stack([noise.standard_normal(5, j, np.arange(mesh.n_dofs)) for j in range(2)])
    assert np.array_equal(W, z * np.sqrt(ML)[None, :])
    # SPEC S253: lumped diag (0.25, 1.0), xi = (2, 3) -> W = (1.0, 3.0)
    assert np.array_equal(np.sqrt(np.array([0.25, 1.0])) * np.array([2.0, 3.0]), np.array([1.0, 3.0]))
