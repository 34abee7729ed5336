"""The ctypes binding stubs printed in INTEGRATION.md, executed as written.

INTEGRATION.md shows the binding a maintainer of the reference package would
add (`mselast/_gpu.py`: ms_problem_create / ms_precond_build / ms_pcg_solve,
and the generic entry point for foreign operands).  The code blocks are taken
out of the document, pointed at the in-tree library and run on a small
problem; their results must equal the drop-in package's own.
"""

import re
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def stub_namespace():
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    binding = next(b for b in blocks if "def gpu_operator" in b)
    generic = next(b for b in blocks if "def gpu_pcg_any" in b)
    lib = ROOT / "paper_2006_13387_b200" / "libmsgpu.so"
    binding = binding.replace('C.CDLL("libmsgpu.so")', f'C.CDLL("{lib}")')
    ns = {}
    exec(compile(binding, "INTEGRATION.md:binding", "exec"), ns)
    exec(compile(generic, "INTEGRATION.md:generic", "exec"), ns)
    return ns


def test_integration_stubs_run_and_match_the_package():
    import paper_2006_13387_b200 as G

    ns = stub_namespace()
    assert ns["lib"].ms_abi_version() == 4
    mesh = G.build_fine_mesh(40, 40)
    part = G.build_coarse_partition(mesh, 4, 4)
    rng = np.random.default_rng(3)
    E = np.where(rng.random(mesh.n_elements) < 0.3, 1.0, 1e-4)
    coeff = G.CoefficientField(E, 0.3, 1e-4, 1.0)
    dn = mesh.boundary_nodes()
    op = G.assemble_elasticity(mesh, coeff, dn)
    pre = G.build_preconditioner("EH+Rot", op, mesh, part, coeff, dn)
    b = rng.standard_normal(op.n_free)
    x_pkg, rep = G.pcg_solve(op, b, pre, tol=1e-8, maxit=500)
    assert rep.converged
    # the stub's own handles: same operator, same preconditioner, same solve
    h = ns["gpu_operator"](mesh, coeff, op.free_dofs)
    pc = ns["gpu_preconditioner"](h, part, dn, "EH+Rot")
    x_stub = ns["gpu_pcg"](h, pc, b, 1e-8, 500)
    assert np.array_equal(x_stub, x_pkg)
    # foreign operands through the generic entry point: scipy CSR + a Python preconditioner
    K = op.matrix.tocsr()
    x_any = ns["gpu_pcg_any"](K, pre.apply, b, 1e-8, 500)
    assert np.linalg.norm(x_any - x_pkg) <= 1e-7 * np.linalg.norm(x_pkg)
    dinv = 1.0 / K.diagonal()
    x_jac = ns["gpu_pcg_any"](sp.csr_matrix(K), lambda r: dinv * r, b, 1e-8, 5000)
    assert np.linalg.norm(K @ x_jac - b) <= 2e-8 * np.linalg.norm(b)
    ns["lib"].ms_precond_destroy(pc)
    ns["lib"].ms_problem_destroy(h)
