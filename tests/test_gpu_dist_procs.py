"""The multi-GPU product path (DistH2Matrix -> igb_h2_create_dist /
igb_h2_dist_phase1 / igb_h2_dist_phase2) run as real separate processes:
world 2 and 3, one rank per process, all on the single B200 of this
environment, with a gloo process group staging the two exchanges (all-gather
of the up moments, all-reduce of y) through host memory -- so no kernel ever
waits on another rank's kernel.  The result must equal the single-GPU matvec."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pde(igb, kind):
    if kind == "laplace":
        return igb.Pde.laplace()
    return igb.Pde.helmholtz(3.0) if kind == "helmholtz" else igb.Pde.maxwell(3.0)


def _worker(rank, world, port, case, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1906_00785_b200 as igb

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    kind, P, rep, L, m = case
    d = igb.Discretization(igb.make_sphere(), _pde(igb, kind), P, rep, L)
    D = igb.DistH2Matrix(d, igb.H2Options(m=m, eta=1.6), device=0)
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, d.dof_count())
    if D.dtype == torch.complex128:
        x = x + 1j * rng.uniform(-1, 1, d.dof_count())
    xd = torch.from_numpy(x).to(D.dtype).cuda()
    y = D.apply(xd)
    y2 = D.apply(xd)  # graphs already instantiated: the steady-state path
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"y{rank}.npy"), y.cpu().numpy())
    np.save(os.path.join(outdir, f"yy{rank}.npy"), y2.cpu().numpy())
    np.save(os.path.join(outdir, f"near{rank}.npy"), np.array(D.h.device_bytes()["near"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [("laplace", 3, 1, 3, 4), ("laplace", 4, 1, 3, 5), ("helmholtz", 2, 1, 2, 6),
                                  ("maxwell", 2, 1, 2, 4)], ids=lambda c: "-".join(map(str, c)))
def test_dist_processes_match_single_gpu(igb, case, world, tmp_path):
    import torch.multiprocessing as mp
    kind, P, rep, L, m = case
    d = igb.Discretization(igb.make_sphere(), _pde(igb, kind), P, rep, L)
    full = igb.H2Matrix(d, igb.H2Options(m=m, eta=1.6), stored_couplings=False)
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, d.dof_count())
    if full.dtype == np.complex128:
        x = x + 1j * rng.uniform(-1, 1, d.dof_count())
    y_ref = full.apply(x)
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ys = [np.load(tmp_path / f"y{r}.npy") for r in range(world)]
    for r in range(world):
        assert np.linalg.norm(ys[r] - y_ref) / np.linalg.norm(y_ref) < 1e-13
        assert np.array_equal(ys[r], ys[0])  # replicated result
        assert np.array_equal(np.load(tmp_path / f"yy{r}.npy"), ys[r])  # deterministic
    near = sum(int(np.load(tmp_path / f"near{r}.npy")) for r in range(world))
    assert near == full.device_bytes()["near"]  # block rows split, not replicated
