"""Helpers for the world_size > 1 tests: spawn ranks with a gloo process group."""
import os
import socket
import tempfile
import traceback

import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(rank, world, port, fn, args, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = fn(rank, world, *args)
        import pickle
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
    except Exception:
        with open(os.path.join(outdir, f"r{rank}.err"), "w") as f:
            f.write(traceback.format_exc())
        raise
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world, *args, timeout=600):
    """Run fn(rank, world, *args) in `world` spawned processes; return the per-rank results."""
    import pickle
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        port = free_port()
        procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, d)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout)
        errs = [open(os.path.join(d, f)).read() for f in sorted(os.listdir(d)) if f.endswith(".err")]
        if errs:
            raise AssertionError("rank failed:\n" + "\n".join(errs))
        for p in procs:
            if p.exitcode != 0:
                raise AssertionError(f"rank exited with {p.exitcode}")
        return [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(world)]
