"""Serialised phase times of rank 0's matvec at world 2 / 4 / 8 (c2, one GPU;
the all-gathered moments are left zero -- timing only)."""
import sys
sys.path.insert(0, ".")
import paper_1906_00785_b200 as igb
d = igb.Discretization(igb.make_sphere(), igb.Pde.laplace(), 3, 1, 6)
for world in (1, 2, 4, 8):
    h = igb.H2Matrix(d, igb.H2Options(m=4), world=world, rank=0)
    p = h.profile_apply(20)
    p = h.profile_apply(50)
    print(world, {k: round(v / 50, 4) for k, v in p.items()}, "sum", round(sum(p.values()) / 50, 4))
    del h
