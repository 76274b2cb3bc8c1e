"""Spectra on the GPU (paper_2507_02809_b200/spectra.py): the reference's own
test_spectra.cpp cases — dense assembly against the matrix-free apply and the oracle's realisation,
the block structure of P, the cap, simple eigenvalue / condition-number identities, and the
reference condition numbers at n = S = 16 (Table 1: 2021.13 and 62.31)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
F = pytest.importorskip("paper_2507_02809_b200.fracinv")
from paper_2507_02809_b200 import spectra as SP  # noqa: E402
from oracle import fracinv_oracle as O  # noqa: E402


def paper(M, beta, omega, n, S):
    return M.make_problem("paper1d", beta, omega, [n], S, 5e-3, 0.01)


def test_dense_assembly_matches_matrix_free_apply():
    A = F.SystemOperator(paper(F, 0.5, 1.5, 8, 4))
    M = SP.assemble_dense_system(A, SP.SYSTEM_A).cpu().numpy()
    for j in range(A.dim()):
        u = np.zeros(A.dim())
        u[j] = 1.0
        col = A.apply(u)
        assert np.abs(M[:, j] - col).max() <= 1e-14 * max(1.0, np.abs(col).max())


@pytest.mark.parametrize("kind", [SP.SYSTEM_A, SP.PRECONDITIONER_P, SP.FORWARD_AHAT])
@pytest.mark.parametrize("case", ["paper", "2d"])
def test_dense_assembly_is_the_reference_realisation(kind, case):
    """The oracle's restatement of spectra.cpp:14-45 (same operation order): bit-for-bit in 1D."""
    if case == "paper":
        spec_f, spec_o = paper(F, 0.1, 1.9, 16, 16), paper(O, 0.1, 1.9, 16, 16)
    else:
        spec_f = F.make_problem("constant", 0.5, 1.5, [5, 5], 8, 5e-3, 0.01)
        spec_o = O.make_problem("constant", 0.5, 1.5, [5, 5], 8, 5e-3, 0.01)
    M = SP.assemble_dense_system(F.SystemOperator(spec_f), kind).cpu().numpy()
    Mo = O.assemble_dense_system(O.SystemOperator(spec_o), kind)
    if case == "paper":
        assert np.array_equal(M, Mo)
    else:  # the 2D generating tensors themselves differ in the last bits (direct cosine sums vs the
        # oracle's FFT of the same rectangle rule), the assembly does not add any difference
        assert np.abs(M - Mo).max() <= 1e-14 * np.abs(Mo).max()


def test_preconditioner_assembly_zeroes_the_trailing_block_column():
    n, S = 6, 3
    A = F.SystemOperator(paper(F, 0.1, 1.9, n, S))
    Ad = SP.assemble_dense_system(A, SP.SYSTEM_A).cpu().numpy()
    Pd = SP.assemble_dense_system(A, SP.PRECONDITIONER_P).cpu().numpy()
    assert np.linalg.norm(Pd[: S * n, S * n:]) == 0.0
    diff = Ad - Pd
    diff[: S * n, S * n:] = 0.0
    assert np.linalg.norm(diff) == 0.0
    Fd = SP.assemble_dense_system(A, SP.FORWARD_AHAT).cpu().numpy()
    assert np.linalg.norm(Pd[: S * n, : S * n] - Fd) == 0.0


def test_assembly_respects_the_dense_cap():
    A = F.SystemOperator(paper(F, 0.5, 1.5, 16, 16))
    with pytest.raises(F.ResourceLimitError):
        SP.assemble_dense_system(A, SP.SYSTEM_A, 64)


def test_eigenvalues_and_condition_numbers_of_simple_matrices():
    assert np.all(np.abs(SP.eigenvalues_dense(np.eye(5)) - 1.0) <= 1e-14)
    ev = np.sort_complex(SP.eigenvalues_dense(np.diag([1.0, 2.0, 3.0])))
    assert list(ev) == [1.0, 2.0, 3.0]
    M = np.random.default_rng(19).uniform(-1, 1, (50, 50))
    assert abs(SP.eigenvalues_dense(M).sum() - np.trace(M)) <= 1e-8 * abs(np.trace(M))
    assert SP.condition_number_2(np.eye(4)) == pytest.approx(1.0)
    assert SP.condition_number_2(np.diag([10.0, 1.0])) == pytest.approx(10.0, rel=1e-12)
    assert np.isinf(SP.condition_number_2(np.zeros((3, 3))))


def test_reference_condition_numbers_n16_S16():
    """test_spectra.cpp:82-88 (the paper's Table 1 cell)."""
    A = F.SystemOperator(paper(F, 0.1, 1.9, 16, 16))
    Ad = SP.assemble_dense_system(A, SP.SYSTEM_A)
    Pd = SP.assemble_dense_system(A, SP.PRECONDITIONER_P)
    assert SP.condition_number_2(Ad) == pytest.approx(2021.13, rel=1e-4)
    assert SP.condition_number_preconditioned(Pd, Ad) == pytest.approx(62.31, rel=1e-4)


@pytest.mark.parametrize("beta,omega", [(0.1, 1.9), (0.5, 1.5), (0.9, 1.1)])
def test_preconditioning_lowers_the_condition_number(beta, omega):
    A = F.SystemOperator(paper(F, beta, omega, 16, 16))
    Ad = SP.assemble_dense_system(A, SP.SYSTEM_A)
    Pd = SP.assemble_dense_system(A, SP.PRECONDITIONER_P)
    assert SP.condition_number_preconditioned(Pd, Ad) < SP.condition_number_2(Ad)


def test_spectral_summary_counts_the_cluster_at_one():
    import torch
    n, S = 16, 8
    A = F.SystemOperator(paper(F, 0.1, 1.9, n, S))
    Ad = SP.assemble_dense_system(A, SP.SYSTEM_A)
    Pd = SP.assemble_dense_system(A, SP.PRECONDITIONER_P)
    s = SP.spectral_summary(torch.linalg.solve(Pd, Ad))
    assert s.cluster_count + s.outlier_count == (S + 1) * n
    assert s.cluster_count >= S * n and s.outlier_count <= n and s.cond_2 > 1.0


def test_preconditioner_is_a_rank_N_correction_with_a_cluster_at_one():
    """test_krylov.cpp:184-202 — also the structural fact the split Arnoldi step rests on (A - P is
    the f column of the time rows only)."""
    import torch
    N, S = 16, 8
    A = F.SystemOperator(paper(F, 0.1, 1.9, N, S))
    Ad = SP.assemble_dense_system(A, SP.SYSTEM_A)
    Pd = SP.assemble_dense_system(A, SP.PRECONDITIONER_P)
    sv = torch.linalg.svdvals(Ad - Pd).cpu().numpy()
    assert int((sv > 1e-10 * sv[0]).sum()) <= N
    ev = SP.eigenvalues_preconditioned(Pd, Ad)
    assert int((np.abs(ev - 1.0) <= 1e-6).sum()) >= S * N


@pytest.mark.parametrize("S", [8, 16])
def test_preconditioned_iterations_bounded_by_N_plus_1(S):
    """test_krylov.cpp:204-216 (reference GMRES settings: full GMRES, tol 1e-8)."""
    A = F.SystemOperator(paper(F, 0.5, 1.5, 16, S))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, F.add_noise(F.forward_solve(A, P).mu, 0.01, 1)).z
    _, rep = F.gmres(A, P, z)
    assert rep.converged and rep.iterations <= 17


def test_concurrent_contexts_are_bitwise_identical():
    """test_toeplitz.cpp:123-143: two host threads, each with its own context (stream and
    workspaces), apply operators of the same problem 50 times; the results equal a serial apply
    bit for bit."""
    import threading
    spec = paper(F, 0.3, 1.3, 64, 16)
    ops = [F.SystemOperator(spec, ctx=F.Context(0)) for _ in range(2)]
    rng = np.random.default_rng(3)
    xs = [rng.uniform(-1, 1, ops[0].dim()) for _ in range(2)]
    ref = [ops[k].apply(xs[k]) for k in range(2)]
    out = [None, None]

    def work(k):
        for _ in range(50):
            out[k] = ops[k].apply(xs[k])

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(2):
        assert np.array_equal(out[k], ref[k])
