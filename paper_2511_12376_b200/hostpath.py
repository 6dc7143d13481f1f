"""Host-memory codec path: pinned host buffers in, pinned host buffers out.

This is what the reference-facing API costs end to end when the tensors live
in host memory (the reference's `TensorBlob` holds host bytes).  The tensor is
cut into 8192-aligned chunks that flow through a ring of CUDA streams so that
H2D copies, the sm_100a kernels and D2H copies of neighbouring chunks overlap:

    encode: H2D(base_i, cur_i) -> bsnp_delta_encode(chunk i) -> D2H(mask_i)
            ... then D2H of each chunk's payload at its exclusive prefix
    decode: H2D(base_i, mask_i, payload_i) -> bsnp_delta_decode -> D2H(out_i)

Chunked encoding is exact: chunk starts are multiples of 8, so each chunk's
mask is a contiguous slice of the whole mask and the payloads concatenate in
element order (bitmask.py:102-103).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _runtime as rt
from . import bitmask as B

CHUNK = 1 << 25  # elements per chunk (64 MiB of 16-bit data), multiple of 8192


@dataclass
class HostDeltaRecord:
    mask: torch.Tensor          # pinned u8 [ceil(n/8)]
    payload: torch.Tensor       # pinned int16 [n_c]
    n: int
    n_c: int
    chunk_counts: list          # n_c per chunk (derivable from the mask)


class HostDeltaCodec:
    def __init__(self, device: torch.device, n: int, chunk: int = CHUNK, streams: int = 3):
        self.dev = device
        self.n = n
        self.chunk = chunk
        self.nchunks = max(1, (n + chunk - 1) // chunk)
        self.streams = [torch.cuda.Stream(device) for _ in range(streams)]
        self.b_d = torch.empty(n, dtype=torch.int16, device=device)
        self.c_d = torch.empty(n, dtype=torch.int16, device=device)
        self.m_d = torch.empty((n + 7) // 8, dtype=torch.uint8, device=device)
        self.p_d = torch.empty(n, dtype=torch.int16, device=device)
        self.st = rt.new_status(device, self.nchunks)
        self.mask_h = torch.empty((n + 7) // 8, dtype=torch.uint8, pin_memory=True)
        self.payload_h = torch.empty(n, dtype=torch.int16, pin_memory=True)
        self.out_h = torch.empty(n, dtype=torch.int16, pin_memory=True)

    def _ranges(self):
        for i in range(self.nchunks):
            s = i * self.chunk
            yield i, s, min(self.n, s + self.chunk)

    def encode(self, base_h: torch.Tensor, cur_h: torch.Tensor) -> HostDeltaRecord:
        base_h, cur_h = base_h.view(torch.int16), cur_h.view(torch.int16)
        main = torch.cuda.current_stream(self.dev)
        for s in self.streams:
            s.wait_stream(main)
        for i, a, b in self._ranges():
            s = self.streams[i % len(self.streams)]
            with torch.cuda.stream(s):
                self.b_d[a:b].copy_(base_h[a:b], non_blocking=True)
                self.c_d[a:b].copy_(cur_h[a:b], non_blocking=True)
                B.encode_delta_async(self.b_d[a:b], self.c_d[a:b], self.m_d[a // 8:(b + 7) // 8],
                                     self.p_d[a:b], self.st[i])
                self.mask_h[a // 8:(b + 7) // 8].copy_(self.m_d[a // 8:(b + 7) // 8],
                                                       non_blocking=True)
        for s in self.streams:
            main.wait_stream(s)
        counts = [c for c, _ in rt.read_status(self.st)]   # one sync
        off = 0
        for i, a, b in self._ranges():
            c = counts[i]
            if c:
                s = self.streams[i % len(self.streams)]
                s.wait_stream(main)
                with torch.cuda.stream(s):
                    self.payload_h[off:off + c].copy_(self.p_d[a:a + c], non_blocking=True)
            off += c
        for s in self.streams:
            s.synchronize()
        return HostDeltaRecord(self.mask_h, self.payload_h[:off], self.n, off, counts)

    def decode(self, base_h: torch.Tensor, rec: HostDeltaRecord) -> torch.Tensor:
        base_h = base_h.view(torch.int16)
        counts = rec.chunk_counts
        if counts is None:
            m = rec.mask.numpy()
            counts = [int(np.bitwise_count(m[a // 8:(b + 7) // 8]).sum())
                      for _, a, b in self._ranges()]
        main = torch.cuda.current_stream(self.dev)
        for s in self.streams:
            s.wait_stream(main)
        off = 0
        for i, a, b in self._ranges():
            s = self.streams[i % len(self.streams)]
            c = counts[i]
            with torch.cuda.stream(s):
                self.b_d[a:b].copy_(base_h[a:b], non_blocking=True)
                self.m_d[a // 8:(b + 7) // 8].copy_(rec.mask[a // 8:(b + 7) // 8],
                                                    non_blocking=True)
                if c:
                    self.p_d[a:a + c].copy_(rec.payload[off:off + c], non_blocking=True)
                B.decode_delta_async(self.b_d[a:b], self.m_d[a // 8:(b + 7) // 8],
                                     self.p_d[a:a + c], c, self.c_d[a:b], self.st[i])
                self.out_h[a:b].copy_(self.c_d[a:b], non_blocking=True)
            off += c
        for s in self.streams:
            main.wait_stream(s)
        res = rt.read_status(self.st)
        for (pc, flags), c in zip(res, counts):
            B._raise_decode_flags(flags, pc, c)
        return self.out_h

    def roundtrip(self, base_h: torch.Tensor, cur_h: torch.Tensor, lag: int = 4):
        """Save + restore of one delta checkpoint through pinned host memory:
        H2D of base and current once, encode, D2H of the record (mask +
        payload), decode of that record onto the device copy of the base
        (the previous checkpoint stays resident, as in chain replay,
        store.py:441-454), D2H of the restored tensor.  Chunk i's decode is
        issued `lag` chunks behind its encode on separate streams, so the
        H2D copies of later chunks overlap the D2H copies of earlier ones;
        the host learns each chunk's n_c from that chunk's event.
        Returns (HostDeltaRecord, restored pinned tensor)."""
        base_h, cur_h = base_h.view(torch.int16), cur_h.view(torch.int16)
        main = torch.cuda.current_stream(self.dev)
        if not hasattr(self, "dstreams"):
            self.dstreams = [torch.cuda.Stream(self.dev) for _ in range(2)]
            self.st_h = torch.empty((self.nchunks, 2), dtype=torch.int64, pin_memory=True)
            self.dst = rt.new_status(self.dev, self.nchunks)
        st_h, dst = self.st_h, self.dst
        for s in self.streams + self.dstreams:
            s.wait_stream(main)
        ranges = list(self._ranges())
        events, counts = [None] * self.nchunks, [0] * self.nchunks
        offs = [0] * (self.nchunks + 1)

        def encode(i, a, b):
            s = self.streams[i % len(self.streams)]
            with torch.cuda.stream(s):
                self.b_d[a:b].copy_(base_h[a:b], non_blocking=True)
                self.c_d[a:b].copy_(cur_h[a:b], non_blocking=True)
                B.encode_delta_async(self.b_d[a:b], self.c_d[a:b], self.m_d[a // 8:(b + 7) // 8],
                                     self.p_d[a:b], self.st[i])
                st_h[i].copy_(self.st[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                events[i] = ev

        def finish(i, a, b):
            events[i].synchronize()
            c, flags = int(st_h[i, 0]), int(st_h[i, 1])
            if flags:
                raise B.DeltaError("internal: payload capacity exceeded")
            counts[i] = c
            offs[i + 1] = offs[i] + c
            s = self.dstreams[i % len(self.dstreams)]
            s.wait_event(events[i])
            with torch.cuda.stream(s):
                self.mask_h[a // 8:(b + 7) // 8].copy_(self.m_d[a // 8:(b + 7) // 8],
                                                       non_blocking=True)
                if c:
                    self.payload_h[offs[i]:offs[i] + c].copy_(self.p_d[a:a + c],
                                                              non_blocking=True)
                B.decode_delta_async(self.b_d[a:b], self.m_d[a // 8:(b + 7) // 8],
                                     self.p_d[a:a + c], c, self.c_d[a:b], dst[i])
                self.out_h[a:b].copy_(self.c_d[a:b], non_blocking=True)

        for i, a, b in ranges:
            encode(i, a, b)
            if i >= lag:
                finish(*ranges[i - lag])
        for i, a, b in ranges[max(0, self.nchunks - lag):]:
            finish(i, a, b)
        for s in self.streams + self.dstreams:
            main.wait_stream(s)
        for (pc, flags), c in zip(rt.read_status(dst), counts):
            B._raise_decode_flags(flags, pc, c)
        rec = HostDeltaRecord(self.mask_h, self.payload_h[:offs[-1]], self.n, offs[-1], counts)
        return rec, self.out_h
