import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2605_11111_b200 as m
DEV="cuda"
torch.manual_seed(0)
shape, cout, R, fmt, dim = (1, 16, 256, 256, 256), 32, 8, torch.channels_last_3d, 2
w = (torch.randn(cout, 16, 3, 3, 3, device=DEV) * 0.05).to(torch.bfloat16)
x = torch.randn(shape, device=DEV).to(torch.bfloat16).contiguous(memory_format=fmt)
dense = m.dense_conv(x, w, stride=1, padding=1)
dense2 = m.dense_conv(x, w, stride=1, padding=1)
print("dense deterministic:", torch.equal(dense, dense2))
ext = m.default_chunk(256, R)
def prog(ctx):
    lo = sum(ext[:ctx.rank_id])
    xl = x.narrow(dim, lo, ext[ctx.rank_id]).contiguous(memory_format=fmt)
    st = m.ShardTensor(xl, tuple(x.shape), ctx, (m.Shard(dim),), {0: tuple(ext)})
    out, tape = m.halo_conv_forward(st, w, 1, 1)
    return out.full_tensor(), out.shard_shapes[0]
full, shapes = m.spawn_mesh((R,), ("domain",), prog)[0]
print(shapes)
d = (full.float() - dense.float()).abs()
rows = d.amax(dim=(0, 1, 3, 4))
bad = (rows > 0).nonzero().flatten().tolist()
print("rows differing along D:", bad[:40], len(bad), "max", d.max().item())
dq = d.amax(dim=(0, 1, 2, 4)); print("H rows differing:", (dq > 0).nonzero().flatten().tolist()[:20], int((dq>0).sum()))
dw_ = d.amax(dim=(0, 1, 2, 3)); print("W cols differing:", (dw_ > 0).nonzero().flatten().tolist()[:20], int((dw_>0).sum()))
frac = (d > 0).float().mean().item(); print("fraction differing", frac)
