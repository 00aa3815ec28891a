"""Frame ingest and mask egress around the device engine (SURVEY.md 8(f)
row 2; reference call path: cli.cmd_run -> load_sequence -> process_frame
-> write_mask, cogbg/cli.py:103-129, cogbg/frame_io.py:231-275).

The reference decodes, steps and writes one frame at a time on one core.
Here the three stages overlap:

  decode   a thread pool decodes image files (Pillow releases the GIL in
           its codecs) up to ``prefetch`` frames ahead, in index order;
  step     ``engine.process_frame`` copies each frame into the engine's
           pinned staging ring and enqueues H2D -> step -> D2H without
           blocking;
  egress   results are read ``lag`` frames behind the submission point (so
           the device->host copies overlap later steps) and handed to the
           callback / written as PNG masks by a writer pool.
"""

from __future__ import annotations

import concurrent.futures as cf
from collections import deque
from pathlib import Path
from typing import Callable, Iterator

import numpy as np

from .frame_io import (LabelMask, SequenceManifest, decode_frame,
                       discover_frame_count, write_mask)


def prefetch_frames(manifest: SequenceManifest, start: int, stop: int,
                    color: bool = False, prefetch: int = 8,
                    workers: int = 4) -> Iterator[tuple[int, np.ndarray]]:
    """(index, (d, H, W) uint8) for frames [start, stop), decoded ahead on
    ``workers`` threads, yielded in index order."""
    with cf.ThreadPoolExecutor(workers) as pool:
        futs: deque = deque()
        nxt = start
        shape = None
        while nxt < stop or futs:
            while nxt < stop and len(futs) < prefetch:
                futs.append((nxt, pool.submit(
                    decode_frame, manifest.frame_path(nxt), nxt, color)))
                nxt += 1
            i, fut = futs.popleft()
            arr = fut.result()
            if shape is None:
                shape = arr.shape
            elif arr.shape != shape:
                from .errors import FormatError
                raise FormatError(f"frame {i} geometry {arr.shape} != first "
                                  f"frame {shape}")
            yield i, arr


def run_stream(engine, frames, on_result: Callable | None = None,
               lag: int = 2) -> int:
    """Push (index, frame) pairs through ``engine.process_frame``; each
    result (index, LabelMask, FrameStats) is read ``lag`` frames later and
    passed to ``on_result``.  Returns the number of frames processed."""
    pending: deque = deque()
    n = 0
    for i, arr in frames:
        m, st = engine.process_frame(arr)
        pending.append((i, m, st))
        n += 1
        while len(pending) > lag:
            j, mj, sj = pending.popleft()
            mj.labels  # noqa: B018 -- wait for this frame's copies
            if on_result is not None:
                on_result(j, mj, sj)
    while pending:
        j, mj, sj = pending.popleft()
        mj.labels  # noqa: B018
        if on_result is not None:
            on_result(j, mj, sj)
    return n


def run_manifest(engine, manifest: SequenceManifest, out_dir=None,
                 start: int | None = None, stop: int | None = None,
                 color: bool | None = None, prefetch: int = 8,
                 workers: int = 4, on_result: Callable | None = None) -> list:
    """Process a manifest's frames [start, stop) (default: everything after
    the training frames), writing ``mask_%06d.png`` into ``out_dir`` when
    given.  Returns the per-frame statistics rows."""
    total = discover_frame_count(manifest)
    start = manifest.training_count if start is None else start
    stop = total if stop is None else min(stop, total)
    color = engine.depth == 3 if color is None else color
    rows: list = []
    out = Path(out_dir) if out_dir is not None else None
    with cf.ThreadPoolExecutor(workers) as writers:
        jobs = []

        def done(i: int, m: LabelMask, st) -> None:
            rows.append(st.as_row())
            if out is not None:
                jobs.append(writers.submit(write_mask, LabelMask(m.labels),
                                           out / f"mask_{i:06d}.png"))
            if on_result is not None:
                on_result(i, m, st)

        run_stream(engine, prefetch_frames(manifest, start, stop, color,
                                           prefetch, workers), done)
        for j in jobs:
            j.result()
    return rows
