"""Multi-rank (strip-sharded) path.

CPU: world_size-2 gloo process groups check that the C++ strip partition and
halo plans (the exact functions the solver uses, via the ABI, no CUDA) pair
up across ranks.  GPU: two ranks on the single available B200 talk through
gloo host callbacks (their kernels never wait on each other) and must
reproduce the one-rank solve.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ---------------------------------------------------------------------------
# CPU: partition and halo pairing


def _plan_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    from paper_2006_13387_b200 import dist as D

    _init(rank, world, port)
    try:
        out = {}
        for nrows, H, ny, k in ((4, 16, 64, 2), (7, 32, 224, 3), (64, 32, 2048, 2)):
            lo, hi = D.strip_rows(nrows, world, rank)
            b_lo = lo * H
            b_hi = ny if hi == nrows else hi * H - 1
            plan = D.halo_plan(b_lo, b_hi, ny, k, rank, world)
            allp = [None] * world
            dist.all_gather_object(allp, (lo, hi, b_lo, b_hi, plan))
            out[(nrows, H, ny, k)] = allp
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_partition_and_halo_pairing_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for key, allp in res[0].items():
        nrows, H, ny, k = key
        # every rank saw the same plans
        assert all(res[r][key] == allp for r in range(world))
        # strips tile [0, nrows) and node rows tile [0, ny]
        assert allp[0][0] == 0 and allp[-1][1] == nrows
        assert all(allp[r][1] == allp[r + 1][0] for r in range(world - 1))
        assert allp[0][2] == 0 and allp[-1][3] == ny
        assert all(allp[r][3] + 1 == allp[r + 1][2] for r in range(world - 1))
        # every send matches the partner's receive (rows and counts)
        for r in range(world):
            for slot in (0, 1):
                s_lo, s_n, dst, _, _, _ = allp[r][4][slot]
                if dst < 0:
                    assert s_n == 0
                    continue
                _, _, _, r_lo, r_n, src = allp[dst][4][slot]
                assert src == r and r_lo == s_lo and r_n == s_n and s_n == min(k, allp[r][3] - allp[r][2] + 1)


# ---------------------------------------------------------------------------
# GPU: 2 ranks on one device through gloo host callbacks


def _solve_worker(rank, world, port, q, tag="EH+Rot"):
    sys.path.insert(0, str(ROOT))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _init(rank, world, port)
    try:
        from paper_2006_13387_b200 import configs, dist as D, pcg_solve
        from paper_2006_13387_b200.solve import setup_spec

        D.init_host_callbacks(0)
        spec = configs.config1(seed=0)
        mesh, op, pre = setup_spec(spec, tag)
        x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=5000)
        z = pre.apply(np.linspace(-1.0, 1.0, op.n_free))
        q.put((rank, x, rep.iterations, rep.converged, pre.coarse_dim, list(pre.mode_counts), z))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["EH+Rot", "HH+Rot", "EE", "EH+Rot;Rand"])
def test_two_ranks_on_one_gpu_match_single_rank(tag):
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_solve_worker, args=(r, 2, port, q, tag)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((v[0], v[1:]) for v in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sys.path.insert(0, str(ROOT))
    from paper_2006_13387_b200 import configs, pcg_solve
    from paper_2006_13387_b200.solve import setup_spec

    spec = configs.config1(seed=0)
    mesh, op, pre = setup_spec(spec, tag)
    x1, rep1 = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=5000)
    z1 = pre.apply(np.linspace(-1.0, 1.0, op.n_free))
    # the reference's own solve of this config and its measured round-off band
    # (tests/golden/make_golden.py): the sharded solve must sit inside it
    g = np.load(ROOT / "tests" / "golden" / ("ref_config1_hhrot.npz" if tag == "HH+Rot" else "ref_config1.npz"))
    its = np.concatenate([[int(g["iters"])], g["jitter_iters"]])
    ref_variant = tag in ("EH+Rot", "HH+Rot")
    for r in (0, 1):
        x, iters, conv, nc, modes, z = res[r]
        assert conv and nc == pre.coarse_dim and modes == list(pre.mode_counts)
        assert np.linalg.norm(z - z1) <= 1e-12 * np.linalg.norm(z1)
        if ref_variant:
            assert its.min() - 1 <= iters <= its.max() + 1, (iters, its)
            assert np.linalg.norm(x - g["x"]) <= max(1e-8, 2 * g["jitter_x"].max()) * np.linalg.norm(g["x"])
        # only the dot-product and coarse-solve summation orders differ from one rank
        assert np.linalg.norm(x - x1) <= 1e-8 * np.linalg.norm(x1)
    assert np.array_equal(res[0][0], res[1][0])


@pytest.mark.gpu
def test_bench_multi_rank_path_runs():
    """bench.py under torchrun (2 ranks): strip sharding, sharded coarse solve,
    max-over-ranks timing and the JSON line; ranks share the one GPU through
    the host-callback communicator (--comm callbacks)."""
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import json
    import subprocess

    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--comm", "callbacks", "--mesh-n", "256", "--maxit", "16",
           "--e2e-steps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["iterations_per_step"] == 16
    # 16 iterations of a hard solve: the residual norm is not monotone, only finite
    assert d["e2e"]["value"] > 0 and np.isfinite(d["config"]["true_rel_residual"])


@pytest.mark.gpu
def test_nccl_communicator_single_rank_selftest():
    """The NCCL communicator (dlopen, unique id, ncclCommInitRank, allreduce,
    broadcast, grouped send/recv, collectives captured in a CUDA graph) on a
    one-rank communicator: the only NCCL configuration one GPU allows."""
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import ctypes as C

    sys.path.insert(0, str(ROOT))
    from paper_2006_13387_b200 import _lib

    lib = _lib.load()
    ctx = C.c_void_p()
    _lib.check(lib.ms_ctx_create(0, C.byref(ctx)))
    try:
        uid = C.create_string_buffer(128)
        _lib.check(lib.ms_nccl_unique_id(uid))
        _lib.check(lib.ms_ctx_attach_nccl(ctx, 0, 1, uid.raw), ctx)
        out = np.zeros(4)
        _lib.check(lib.ms_comm_selftest(ctx, _lib.dptr(out)), ctx)
        assert out.tolist() == [1.0, 2.0, 7.0, 0.0]
    finally:
        lib.ms_ctx_destroy(ctx)


def _selftest_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    _init(rank, world, port)
    try:
        from paper_2006_13387_b200 import _lib, dist as D

        ctx = D.init_host_callbacks(0)
        out = np.zeros(4)
        _lib.check(_lib.load().ms_comm_selftest(ctx.handle, _lib.dptr(out)), ctx.handle)
        q.put((rank, out.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_callback_communicator_two_rank_selftest():
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_selftest_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert res[r] == [3.0, 4.0, 7.0, float(1 - r)]


def _strip_worker(rank, world, port, q, n, maxit, bitwise=False):
    sys.path.insert(0, str(ROOT))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ["MS_L1_TWIST"] = "1"
    if bitwise:
        os.environ["MS_DIST_BITWISE"] = "1"
    _init(rank, world, port)
    try:
        from paper_2006_13387_b200 import configs, dist as D, pcg_solve
        from paper_2006_13387_b200.solve import setup_spec

        D.init_host_callbacks(0)
        spec = configs.config3(seed=0, n=n)
        mesh, op, pre = setup_spec(spec, "EH+Rot")
        x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-12, maxit=maxit)
        z = pre.apply(np.linspace(-1.0, 1.0, op.n_free))
        q.put((rank, x, rep.iterations, pre.coarse_dim, list(pre.mode_counts), z,
               pre.info["n_subdomains_local"], rep.residuals))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("bitwise", [False, True])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_strip_ranks_on_one_gpu_match_single_rank(world, bitwise, monkeypatch):
    """Config 3's recipe at 256^2 (8 x 8 subdomain rows) sharded into 2, 4 and
    8 strips, the ranks' kernels on the one B200 and their collectives
    through gloo host callbacks: same coarse space on every rank, the
    subdomain rows partitioned, and the same preconditioner and PCG iterates
    as one rank.  Default mode: only the summation order of the dot products
    and of the sharded coarse solve differ (tolerances).  MS_DIST_BITWISE=1:
    dot products from global block slots and a replicated coarse solve --
    the iterates are bit-identical to one rank."""
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    n, maxit = 256, 40
    monkeypatch.setenv("MS_L1_TWIST", "1")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strip_worker, args=(r, world, port, q, n, maxit, bitwise)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((v[0], v[1:]) for v in (q.get(timeout=900) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sys.path.insert(0, str(ROOT))
    from paper_2006_13387_b200 import configs, pcg_solve
    from paper_2006_13387_b200.solve import setup_spec

    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec, "EH+Rot")
    x1, rep1 = pcg_solve(op, spec.rhs(), pre, tol=1e-12, maxit=maxit)
    z1 = pre.apply(np.linspace(-1.0, 1.0, op.n_free))
    owned = [res[r][5] for r in range(world)]
    assert sum(owned) == pre.info["n_subdomains"] and max(owned) - min(owned) <= spec.Nx
    for r in range(world):
        x, iters, nc, modes, z, _, resid = res[r]
        assert nc == pre.coarse_dim and modes == list(pre.mode_counts)
        assert iters == rep1.iterations == maxit
        if bitwise:
            assert np.array_equal(x, x1), np.abs(x - x1).max()
            assert np.array_equal(np.asarray(resid), np.asarray(rep1.residuals))
        else:
            assert np.linalg.norm(x - x1) <= 1e-10 * np.linalg.norm(x1)
            assert np.allclose(resid, rep1.residuals, rtol=1e-9)
        assert np.linalg.norm(z - z1) <= 1e-12 * np.linalg.norm(z1)
        assert np.array_equal(x, res[0][0])


def _apply_before_build_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    _init(rank, world, port)
    try:
        from paper_2006_13387_b200 import ElasticityOperator, CoefficientField, build_fine_mesh, configs, dist as D

        D.init_host_callbacks(0)
        spec = configs.config1(seed=0)
        mesh = build_fine_mesh(spec.nx, spec.ny)
        op = ElasticityOperator(mesh, CoefficientField(spec.E, spec.nu, spec.E_min, spec.E_max), spec.free_dofs())
        v = np.linspace(-1.0, 1.0, op.n_free)
        q.put((rank, op @ v))  # no preconditioner yet: no strip ownership
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_operator_apply_before_any_preconditioner_two_ranks():
    """with a communicator attached, `op @ v` before any
    preconditioner exists (no strip ownership yet) must not index the empty
    row tables; every rank computes all rows and gets the one-rank result."""
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_apply_before_build_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, str(ROOT))
    from paper_2006_13387_b200 import ElasticityOperator, CoefficientField, build_fine_mesh, configs

    spec = configs.config1(seed=0)
    mesh = build_fine_mesh(spec.nx, spec.ny)
    op = ElasticityOperator(mesh, CoefficientField(spec.E, spec.nu, spec.E_min, spec.E_max), spec.free_dofs())
    ref = op @ np.linspace(-1.0, 1.0, op.n_free)
    for r in (0, 1):
        assert np.array_equal(res[r], ref)
