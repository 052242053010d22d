"""CPU oracle for randUTV (Martinsson, Quintana-Ortí, Heavner, arXiv 1703.00998).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_1703_00998_b200``) may import, call, link or execute anything under
``oracle/``.  The only permitted users are ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.

The oracle is a plain, slow, fp64 implementation that follows the paper's
efficient algorithm (Fig. ``fig:randUTV``) step by step.
It shares no code with the CUDA path.  Library primitives used as single
steps: numpy matmul (BLAS dgemm), numpy norms, and LAPACK's SVD
(``scipy.linalg.svd``, the paper's ``svd`` call at PAPER.md:964/971).  Everything
else (Philox, Gaussian transform, Householder reflectors, compact-WY factor,
applications, the blocked driver) is written out here.

Modules
-------
philox      counter-based Philox4x32-10 + uniform/Box-Muller map (the paper's
            ``randn``; RNG choice = DESIGN.md reading R2)
householder unpivoted Householder QR (LAPACK dlarfg convention, reading R3),
            forward compact-WY T factor, right/left applications
small_svd   b x b SVD via LAPACK gesvd
randutv     the blocked driver of Fig. fig:randUTV
rsvd        the randomized SVD of Remark remark:RSVD

Pins (``tests/test_oracle_*.py``): cuRAND's host Philox, LAPACK dgeqrf, the
explicit reflector product, closed forms, the dense Fig. ``fig:randUTVmatlab``
transcription, the Theorem of §5.3, and whole-factorization invariants.
Parity status of every function is listed in DESIGN.md §"Oracle pins"; no
function is "parity unpinned".
"""
from .philox import philox4x32_10, uniforms, gaussian_block  # noqa: F401
from .householder import house, geqr2, larft, unit_lower, apply_right, apply_left_t, thin_q  # noqa: F401
from .small_svd import small_svd  # noqa: F401
from .randutv import randutv  # noqa: F401
from .rsvd import rsvd  # noqa: F401
