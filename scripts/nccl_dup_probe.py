"""Can two ranks share one GPU in an NCCL communicator (library comm layer)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def run(rank, q, uid):
    try:
        torch.cuda.set_device(0)
        from paper_2605_11111_b200 import comm
        c = comm.NcclComm.init(2, rank, uid)
        a = torch.full((1024,), float(rank + 1), device="cuda")
        b = torch.empty_like(a)
        c.allreduce(a, b)
        c.wait(timeout=30)
        q.put((rank, "ok", float(b[0])))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "err", repr(e)[:300]))


if __name__ == "__main__":
    from paper_2605_11111_b200 import comm
    uid = comm.unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=run, args=(r, q, uid)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(2):
        print(q.get(timeout=120))
    for p in ps:
        p.join(30)
