"""Per-rank distributed matvec time (phase 1 + phase 2, collectives excluded)
of rank 0 at world 2 / 4 / 8 on one GPU (c2)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
o = igb.H2Options(m=4)
dev = 0
for world in (2, 4, 8):
    h = igb.H2Matrix(d, o, device=dev, world=world, rank=0)
    n = h.dist_send_count()
    x = torch.rand(d.dof_count(), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    snd = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
    rcv = torch.zeros(max(n, 1) * world, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        h.dist_phase1(x.data_ptr(), snd.data_ptr(), st)
        h.dist_phase2(rcv.data_ptr(), y.data_ptr(), st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        h.dist_phase1(x.data_ptr(), snd.data_ptr(), st)
        h.dist_phase2(rcv.data_ptr(), y.data_ptr(), st)
    b.record()
    torch.cuda.synchronize()
    asm = h.reassemble()[0]
    print(f"world {world}: rank-0 matvec {a.elapsed_time(b) / 100:.4f} ms (collectives excluded), assembly {asm:.2f} ms")
    del h
