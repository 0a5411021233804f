"""Pins of the oracle's SGGX finalisation and 6-byte compact form (docs/PREDICATES.md §11;
SURVEY §8(f) NEXT-3; Eq. compact-sggx): the pinned
Jacobi against LAPACK (numpy.linalg.eigvalsh), the moment-form jitter against a Monte-Carlo
run of SPEC's per-sample jitter, the normalisation against the exact maximum eigenvalue,
and the SPEC encode/decode examples and round-trip bound."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle


def _sym(S6):
    a = np.asarray(S6, np.float64)
    return np.array([[a[0], a[3], a[4]], [a[3], a[1], a[5]], [a[4], a[5], a[2]]])


def _s6(S):
    return [S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]]


def _acc(S):
    return oracle.acc_from_float(1.0, _s6(np.asarray(S, np.float64)))


@pytest.mark.parametrize("seed", range(6))
def test_jacobi_matches_lapack(seed):
    rng = np.random.default_rng(seed)
    Q = Rotation.random(random_state=seed).as_matrix()
    cases = [np.diag(rng.uniform(0, 1, 3)),
             Q @ np.diag(rng.uniform(0, 1, 3)) @ Q.T,
             Q @ np.diag([1.0, 0.0, 0.0]) @ Q.T,                 # rank 1
             Q @ np.diag([0.5, 0.5, 0.0]) @ Q.T,                 # repeated, rank 2
             Q @ np.diag([1.0, 1e-6, 1e-7]) @ Q.T]               # nearly degenerate
    for S in cases:
        S6 = np.asarray(_s6(S), np.float32)
        lam = np.sort(oracle.jacobi(S6).astype(np.float64))
        ref = np.linalg.eigvalsh(_sym(S6))
        assert np.abs(lam - ref).max() <= 4e-7 * max(1.0, np.abs(ref).max()), (S6, lam, ref)


def test_jitter_is_the_moment_of_spec_per_sample_jitter():
    # SPEC jitter_degenerate: every unit direction moved by a uniform offset of magnitude eps,
    # renormalised. Its second moment (Monte Carlo) is what the moment form must reproduce.
    eps = 1e-2
    rng = np.random.default_rng(7)
    for dirs in (np.array([[0.0, 0.0, 1.0]]),                           # all along z (SPEC example)
                 np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]),           # planar, rank 2
                 Rotation.random(random_state=3).apply([[0.0, 0.0, 1.0]])):  # a generic axis
        d = np.repeat(dirs, 1_000_000 // len(dirs), axis=0)          # exact mixture weights
        g = rng.standard_normal(d.shape)
        g /= np.linalg.norm(g, axis=1, keepdims=True)
        d, g = np.concatenate([d, d]), np.concatenate([g, -g])     # antithetic offsets: O(eps) noise cancels
        dp = d + eps * g
        dp /= np.linalg.norm(dp, axis=1, keepdims=True)
        E = dp.T @ dp / len(dp)
        S = dirs.T @ dirs / len(dirs)
        Sn, flag = oracle.finalize(_acc(S))
        assert flag == 1
        En = E / np.linalg.eigvalsh(E).max()
        assert np.abs(_sym(Sn) - En).max() < 3e-6, (_sym(Sn), En)


def test_normalisation_and_threshold():
    Q = Rotation.random(random_state=11).as_matrix()
    for lam, jit in (((1.0, 0.3, 2e-4), 0), ((1.0, 0.3, 5e-5), 1), ((0.6, 0.6, 0.6), 0)):
        S = Q @ np.diag(lam) @ Q.T
        S /= np.trace(S)
        Sn, flag = oracle.finalize(_acc(S))
        assert flag == jit
        assert abs(np.linalg.eigvalsh(_sym(Sn)).max() - 1.0) < 2e-6
    assert oracle.finalize(np.zeros(7, np.int64))[1] == -1


def test_spec_encode_examples():
    # sigma = (1, 0.5, 0.2), r = 0 -> decode within one step (SPEC encode_compact example 1)
    b, jit = oracle.encode(_acc(np.diag([1.0, 0.25, 0.04])))
    assert jit[0] == 0 and b[0].tolist() == [255, 128, 51, 128, 128, 128]
    D = oracle.decode(b)[0]
    assert abs(np.sqrt(D[0, 0]) - 1.0) <= 1 / 255 and abs(np.sqrt(D[1, 1]) - 0.5) <= 1 / 255
    assert abs(np.sqrt(D[2, 2]) - 0.2) <= 1 / 255
    # zero record -> the all-zero-sigma pattern (SPEC example 2)
    b, _ = oracle.encode(np.zeros((1, 7), np.int64))
    assert b[0].tolist() == [0, 0, 0, 128, 128, 128]
    # delta along z (after the mandatory jitter): sigma_z = 1, sigma_x = sigma_y = O(eps), r = 0
    b, jit = oracle.encode(_acc(np.diag([0.0, 0.0, 1.0])))
    assert jit[0] == 1 and b[0, 2] == 255 and b[0, 0] <= 3 and b[0, 1] <= 3 and b[0, 3:].tolist() == [128] * 3


def test_round_trip_random_sggx():
    # 1000 random valid S: every decoded field within one quantisation step, decoded S PSD
    rng = np.random.default_rng(0)
    accs, Sns = [], []
    for t in range(1000):
        Q = Rotation.random(random_state=1000 + t).as_matrix()
        S = Q @ np.diag(rng.dirichlet(np.ones(3))) @ Q.T
        a = _acc(S)
        accs.append(a)
        Sns.append(_sym(oracle.finalize(a)[0]))
    b, _ = oracle.encode(np.stack(accs))
    sg = b[:, :3] / 255.0
    r = b[:, 3:] / 127.5 - 1.0
    for n, Sn in enumerate(Sns):
        want_s = np.sqrt(np.maximum(np.diag(Sn), 0))
        assert np.abs(sg[n] - want_s).max() <= 0.5 / 255 + 1e-6
        for (i, j), c in zip(((0, 1), (0, 2), (1, 2)), range(3)):
            p = Sn[i, i] * Sn[j, j]
            want_r = np.clip(Sn[i, j] / np.sqrt(p), -1, 1) if p > 0 else 0.0
            assert abs(r[n, c] - want_r) <= 0.5 / 127.5 + 1e-6
    D = oracle.decode(b)
    assert np.linalg.eigvalsh(D).min() >= -1e-12
