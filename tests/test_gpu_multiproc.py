"""The row-band decomposition of one stream across PROCESSES (the
multi-GPU path of bench.py --workload c4 --gpus N), run as two ranks over
gloo that share cuda:0: each rank trains its stride-aligned band with
``train_band_engine`` (the grouping features all-gathered with
``dist_gather_rows``) and steps it with the per-frame ``DistReducer``
all-reduce of the exact partials, the host path (process_frame) included.
The union of the ranks' masks, their per-frame statistics and the banded
state must equal the single whole-frame engine bit for bit
(cascade.py:301-317 couplings: group update, illumination, stats).

A second variant sums the partials through peer mailboxes mapped across
the two processes with CUDA IPC (``PeerMailbox.ipc(fused=False)``): the
step's last CTA stores the rank's partials into both ranks' mailboxes
(``cog_step_p2p``), a host barrier follows, ``cog_finalize_p2p`` sums the
own mailbox -- the multi-GPU data path with real cross-process peer stores.

No kernel of one rank waits on the other's on the device (the ranks share
one GPU): the exchange is separated from its consumer by a host-side
all-reduce or barrier between the step and its finalize.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_TRAIN, N_RUN = 30, 24


def _scene():
    from paper_1705_09339_b200 import synth
    spec = synth.small_spec(2, 64, 48, N_TRAIN + N_RUN, N_TRAIN)
    return synth.Scene(spec).frames(0, N_TRAIN + N_RUN)


def _cfg(dtype):
    from paper_1705_09339_b200.config import EngineConfig
    return EngineConfig(k_max=3, color=True, training_frames=N_TRAIN,
                        state_dtype=dtype, chp_epsilon=1.0,
                        saturation_frames=5, sleep_frames=3,
                        reorder_interval=10).validate()


def _rank(rank, world, port, dtype, out_dir, mailbox=False):
    import torch.distributed as dist
    from paper_1705_09339_b200.parallel import (DistReducer, PeerMailbox,
                                                band_rows, dist_gather_rows,
                                                train_band_engine)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    frames = _scene()
    cfg = _cfg(dtype)
    rows = band_rows(frames.shape[2], world, cfg.stride)[rank]
    eng = train_band_engine(frames[:N_TRAIN], cfg, rows,
                            gather=dist_gather_rows())
    if mailbox:
        # the ranks share cuda:0, so the unfused form: push over CUDA IPC
        # peer memory, host barrier, cog_finalize_p2p
        eng.peers = PeerMailbox.ipc(eng.depth, eng.dev.n_groups, fused=False)
    else:
        eng.reducer = DistReducer()
    masks, stats = [], []
    for t in range(N_TRAIN, N_TRAIN + N_RUN):
        m, st = eng.process_frame(np.ascontiguousarray(frames[t][:, rows[0]:rows[1]]))
        masks.append(m.labels.copy())
        stats.append(st.as_row())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), masks=np.stack(masks),
             stats=np.array(stats), mu=eng.mu, var=eng.var, w=eng.w,
             rows=np.array(rows))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mailbox", [False, True])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_two_process_row_bands_equal_single_engine(dtype, mailbox):
    """mailbox=True: the partials cross the process boundary through peer
    mailboxes mapped with CUDA IPC (cog_step_p2p pushes from the step's last
    CTA, cog_finalize_p2p sums) instead of the host all-reduce"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1705_09339_b200.training import train_engine
    world = 2
    with tempfile.TemporaryDirectory() as tmp:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank,
                             args=(r, world, port, dtype, tmp, mailbox))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
            assert p.exitcode == 0, f"rank exited with {p.exitcode}"
        parts = [dict(np.load(os.path.join(tmp, f"rank{r}.npz")))
                 for r in range(world)]
    frames = _scene()
    single = train_engine(frames[:N_TRAIN], _cfg(dtype))
    for i, t in enumerate(range(N_TRAIN, N_TRAIN + N_RUN)):
        m, st = single.process_frame(frames[t])
        want = m.labels
        got = np.concatenate([p["masks"][i] for p in parts], axis=0)
        assert np.array_equal(got, want), f"mask differs at frame {t}"
        row = st.as_row()
        for p in parts:
            assert list(p["stats"][i]) == row, f"stats differ at frame {t}"
    for k in ("mu", "var", "w"):
        got = np.concatenate([p[k] for p in parts], axis=1)
        assert np.array_equal(got, getattr(single, k)), k
