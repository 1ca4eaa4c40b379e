"""Multi-GPU parity (run under torchrun, one rank per GPU -- also with a
single rank, which drives the NCCL code with nranks = 1; launched by
tests/test_gpu_multi.py).  Through the C ABI with an NCCL communicator:
 - even partition: every rank sweeps its contiguous share; the allgather of
   counts gives global offsets, the optional gather gives every rank all
   columns; the collective digest of the sharded result is the digest of the
   global result;
 - cyclic partition (a8, bench.py's default): blocks dealt round-robin
   (me_cyclic_block), swept alone, joined by me_result_join (one NCCL
   allgather + a device scan).
The global result must equal the oracle's single-process result bit for bit."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import me_inputs as mi  # noqa: E402


def main():
    import oracle
    import paper_2411_06465_b200 as me
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    comm = me.Comm(local)
    spaces = [mi.config("C3"), mi.config("C3", uneven=1),
              mi.Space(models=mi.random_models(30, seed=31), world=[24, 96, 1000], caps_gb=[40, 80, 94, 192],
                       mbs=[1, 2, 4], seq=[4096, 8192], uneven=1, gbs=960)]
    ok = True
    for sp in spaces:
        plan = me.Plan(sp, device=local)
        idx, rows, n, caps = oracle.sweep(sp, threads=4) if rank == 0 else (None, None, None, None)
        for k, (begin, end) in enumerate(((0, 0), (7, plan.size - 3))):
            # gathered FULL / RECORDS result on every rank
            r = plan.sweep(begin, end, mode=(me.ME_OUT_FULL, me.ME_OUT_RECORDS)[k], comm=comm, gather=True)
            lo, gl, off = r.counts()
            got = r.to_host()
            # sharded INDEX result: local rows + global offset
            r2 = plan.sweep(begin, end, mode=me.ME_OUT_INDEX, comm=comm)
            lo2, gl2, off2 = r2.counts()
            loc = r2.to_host()["index_mask"]
            parts = [None] * world
            dist.all_gather_object(parts, (off2, loc.tolist()))
            if rank == 0:
                e = end or plan.size
                ridx, rrows, rn, rcaps = oracle.sweep(sp, begin, e, threads=4)
                ok &= gl == rn and gl2 == rn and r.cap_counts() == rcaps
                ok &= np.array_equal(got["index_mask"], ridx)
                for j, k in enumerate(me.TERMS):
                    ok &= np.array_equal(got[k], rrows[:, j])
                cat = []
                for o, l in parts:
                    ok &= o == len(cat)
                    cat += l
                ok &= np.array_equal(np.array(cat, dtype=np.uint64), ridx)
            # the collective rank of the sharded result = the gathered result's
            if len(sp.cap_bytes) >= 2:
                top_sharded = r2.rank(green_cap=0, yellow_cap=1, gpus_per_node=8, k=3)
                top_gathered = r.rank(green_cap=0, yellow_cap=1, gpus_per_node=8, k=3)
                ok &= top_sharded == top_gathered
            # the collective digest of the sharded result = the global result's
            dg = r2.digest()
            if rank == 0:
                ok &= dg == (oracle.digest_of_rows(ridx, rrows)[0], 0)
                ok &= r.digest() == oracle.digest_of_rows(ridx, rrows)
            r.free()
            r2.free()
            # cyclic deal of blocks + one deferred join (block = the whole
            # range: ranks > 0 hold no block and join with n = 0)
            for block in (1000, 7777, 1 << 40):
                e = end or plan.size
                blocks, nb = me.cyclic_blocks(begin, e, block, rank, world)
                res = [plan.sweep(lo_, hi_, mode=me.ME_OUT_RECORDS, partition=me.ME_PART_CYCLIC) for lo_, hi_ in blocks]
                me.result_join(res, nb, comm)
                mine = []
                for rr in res:
                    lo3, gl3, off3 = rr.counts()
                    mine.append((off3, gl3, rr.cap_counts(), rr.to_host()["index_mask"].tolist()))
                parts = [None] * world
                dist.all_gather_object(parts, mine)
                if rank == 0:
                    ridx, rrows, rn, rcaps = oracle.sweep(sp, begin, e, threads=4)
                    allb = sorted(x for p_ in parts for x in p_)
                    cat = []
                    for off3, gl3, cc3, rows3 in allb:
                        ok &= off3 == len(cat) and gl3 == rn and cc3 == rcaps
                        cat += rows3
                    ok &= np.array_equal(np.array(cat, dtype=np.uint64), ridx)
                for rr in res:
                    rr.free()
        plan.free()
    comm.check()
    flag = torch.tensor([1 if ok else 0], device=f"cuda:{local}")
    dist.broadcast(flag, 0)
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_PARITY", "OK" if flag.item() else "FAIL", flush=True)
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
