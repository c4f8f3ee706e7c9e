"""Virtual-world harness: W hz contexts on ONE GPU (hz_init_virtual), one host thread
and one CUDA stream per rank, running the same per-rank check functions the
multi-process parity worker (tests/mp_parity.py) runs under torchrun.  The contexts
exchange through the product's P2P kernels over each other's pools, so the
multi-piece gathers, the hop groups and the level-local phase protocol of the
W-GPU path run — and are compared bit for bit with the oracle — on the 1-GPU box.
"""

import threading
import traceback

import torch


def run_ranks(hz, group, fn, pool_bytes=96 << 20, device=0, timeout_s=300.0, ranks=None, ctxs=None, devices=None):
    """Run fn(rank, world, ctx) -> list of error strings in one thread per rank (each on
    its own stream, on its context's GPU).  Returns all errors (exceptions included,
    with their rank).  ``ranks``: only these ranks run (the others stay idle);
    ``ctxs``: reuse contexts; ``devices``: rank r on GPU devices[r] (hz_init_virtual_ex)."""
    own = ctxs is None
    if own:
        ctxs = hz.virtual_world(group, device=device, pool_bytes=pool_bytes, devices=devices)
        for c in ctxs:
            c.set_wait_timeout(timeout_s)
    world = len(ctxs)
    errors = {r: [] for r in range(world)}

    def body(r):
        torch.cuda.set_device(ctxs[r].device)
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                errors[r] += fn(r, world, ctxs[r]) or []
            st.synchronize()
        except Exception:   # noqa: BLE001 - reported per rank
            errors[r].append(f"[rank {r}] " + traceback.format_exc())

    threads = [threading.Thread(target=body, args=(r,)) for r in (ranks if ranks is not None else range(world))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for d in sorted({c.device for c in ctxs}):
        torch.cuda.synchronize(d)
    if own:
        for c in ctxs:
            c.close()
    return [f"[rank {r}] {e}" for r in range(world) for e in errors[r]]
