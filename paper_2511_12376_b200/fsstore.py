"""The reference store's save / load entry points over the B200 codec.

`save_checkpoint(cfg, ckpt, prev)` and `load_checkpoint(cfg, iteration)`
(/root/reference/pkg/src/bitsnap/store.py:374-392, 418-474) are the callers
of the hot path: save = the base-refresh policy (decide_kind, store.py:306-
323) + encode_checkpoint (GPU) + commit (store.py:339-371); load = walk the
manifests back to the anchoring base, then ONE `decode_chain` on the GPU
(in-place delta apply, batched dequantize).  The on-disk layout — iter_NNNNNNN
directories holding tensors.bin / manifest.bin / type.txt, the tracker file,
the needs-base marker, the lock file — is the reference's, so either
implementation reads what the other wrote.

Kept deliberately thin: the reference's crash-point hooks (faults.py), inspect
and pruning are store maintenance, not codec work; this module is
the byte sink and source around the device codec.
"""

from __future__ import annotations

import os
import shutil
from dataclasses import dataclass
from pathlib import Path

from filelock import FileLock

from . import faults

TRACKER_NAME = "latest_checkpointed_iteration.txt"
LOCK_NAME = ".lock"
NEEDS_BASE_MARKER = ".needs_base"
DIR_PREFIX = "iter_"
DIR_DIGITS = 7


def _errors():
    from . import store as S
    return S


@dataclass
class StoreConfig:
    """store.py:84-111 (same fields, same MAX_CACHED_ITERATION override)."""

    root: Path
    max_cached_iteration: int = 1
    redundancy_depth: int = 2
    quantizer_clusters: int = 16

    def __post_init__(self):
        self.root = Path(self.root)
        S = _errors()
        if self.effective_max_cached() < 1:
            raise S.StoreError("max_cached_iteration must be >= 1")
        if self.redundancy_depth < 1:
            raise S.StoreError("redundancy depth must be >= 1")

    def effective_max_cached(self) -> int:
        env = os.environ.get("MAX_CACHED_ITERATION")
        return int(env) if env is not None else self.max_cached_iteration

    def tracker_path(self) -> Path:
        return self.root / TRACKER_NAME

    def iter_dir(self, iteration: int) -> Path:
        return self.root / f"{DIR_PREFIX}{iteration:0{DIR_DIGITS}d}"

    def lock(self) -> FileLock:
        return FileLock(str(self.root / LOCK_NAME))


def write_tracker(cfg: StoreConfig, state) -> None:
    """store.py:181-187: `state` (a store.TrackerState) through a temp file
    and an atomic rename."""
    path = cfg.tracker_path()
    tmp = path.with_suffix(".tmp")
    tmp.write_text(f"{state.latest_iteration}\n{state.latest_base_iteration}\n")
    faults.trip("store.tracker.temp-written")
    os.replace(tmp, path)
    faults.trip("store.tracker.renamed")


def read_tracker(cfg: StoreConfig):
    """store.py:190-201 -> store.TrackerState; TrackerError when the file is
    missing or malformed."""
    S = _errors()
    path = cfg.tracker_path()
    if not path.exists():
        raise S.TrackerError(f"tracker file not found at {path}")
    lines = path.read_text().splitlines()
    if len(lines) < 2:
        raise S.TrackerError(f"malformed tracker file at {path}")
    try:
        latest, base = int(lines[0]), int(lines[1])
    except ValueError as exc:
        raise S.TrackerError(f"malformed tracker file at {path}: {exc}") from exc
    return S.TrackerState(latest, base)


def try_read_tracker(cfg: StoreConfig):
    try:
        return read_tracker(cfg)
    except _errors().TrackerError:
        return None


def list_iterations(cfg: StoreConfig) -> list:
    if not cfg.root.exists():
        return []
    out = []
    for p in sorted(cfg.root.iterdir()):
        if p.is_dir() and p.name.startswith(DIR_PREFIX):
            try:
                out.append(int(p.name[len(DIR_PREFIX):]))
            except ValueError:
                continue
    return out


def decide_kind(cfg: StoreConfig, iteration: int) -> str:
    """store.py:306-323: a base, then max_cached_iteration - 1 deltas; a
    failed delta save forces the next save to be a base."""
    S = _errors()
    if (cfg.root / NEEDS_BASE_MARKER).exists():
        return S.KIND_BASE
    tracker = try_read_tracker(cfg)
    if tracker is None:
        return S.KIND_BASE
    since_base = sum(1 for it in list_iterations(cfg) if it >= tracker.latest_base_iteration)
    return S.KIND_BASE if since_base >= cfg.effective_max_cached() else S.KIND_DELTA


def commit(cfg: StoreConfig, manifest, tensors) -> None:
    """store.py:339-371: write one checkpoint directory, then advance the
    tracker, under the store lock.  `tensors` may be bytes or a host uint8
    tensor (the encoder's pinned output, written without a copy)."""
    from .store import write_tensors_bin
    S = _errors()
    cfg.root.mkdir(parents=True, exist_ok=True)
    final_dir = cfg.iter_dir(manifest.iteration)
    tmp_dir = cfg.root / f".tmp_{final_dir.name}"
    with cfg.lock():
        try:
            if tmp_dir.exists():
                shutil.rmtree(tmp_dir)
            tmp_dir.mkdir()
            write_tensors_bin(str(tmp_dir / "tensors.bin"), tensors)
            faults.trip("store.dir.tensors-written")
            (tmp_dir / "manifest.bin").write_bytes(manifest.to_bytes())
            faults.trip("store.dir.manifest-written")
            (tmp_dir / "type.txt").write_text(manifest.kind + "\n")
            faults.trip("store.dir.type-written")
            os.replace(tmp_dir, final_dir)
            faults.trip("store.dir.renamed")
            prev = try_read_tracker(cfg)
            if manifest.kind == S.KIND_BASE:
                base = manifest.iteration
            else:
                base = prev.latest_base_iteration if prev else manifest.base_iteration
            write_tracker(cfg, S.TrackerState(manifest.iteration, base))
            marker = cfg.root / NEEDS_BASE_MARKER
            if manifest.kind == S.KIND_BASE and marker.exists():
                marker.unlink()
        except faults.CrashPoint:
            raise           # a crash leaves whatever it left (the tests inspect it)
        except Exception:
            shutil.rmtree(tmp_dir, ignore_errors=True)
            raise


def save_checkpoint(cfg: StoreConfig, ckpt, prev=None, encoder=None):
    """store.py:374-392 -> CheckpointManifest.

    `encoder`: an optional `store.CheckpointEncoder` that keeps the previous
    model states resident in HBM, so a delta save needs no `prev` (the
    reference's service reloads the previous checkpoint from disk first,
    app.py:62-64)."""
    S = _errors()
    kind = decide_kind(cfg, ckpt.iteration)
    encoder_keeps = encoder is not None and bool(encoder.keep_prev)
    try:
        if encoder is None:
            encoder = S.CheckpointEncoder(clusters=cfg.quantizer_clusters, keep_prev=False)
        elif encoder.clusters != cfg.quantizer_clusters:
            raise S.StoreError(f"encoder uses {encoder.clusters} clusters, the store "
                               f"{cfg.quantizer_clusters}")
        manifest, out = encoder.encode(ckpt, prev, kind)
        commit(cfg, manifest, out)
    except faults.CrashPoint:
        # an injected crash stands for the process dying: whatever the
        # encoder retained may not be on disk
        if encoder_keeps:
            encoder.prev = None
        raise
    except Exception:
        # the reference forces a base after a failed delta.  A resident
        # encoder has already taken the failed checkpoint as its next delta
        # base (or may have, mid-encode), which no committed directory holds,
        # so a failed base save forces a base too, and the encoder forgets it:
        # a later delta can never name an uncommitted base_iteration
        if kind == S.KIND_DELTA or encoder_keeps:
            cfg.root.mkdir(parents=True, exist_ok=True)
            (cfg.root / NEEDS_BASE_MARKER).touch()
        if encoder_keeps:
            encoder.prev = None
        raise
    return manifest


def prune_above(cfg: StoreConfig, iteration: int) -> list:
    """store.py:533-553: remove every checkpoint newer than `iteration` (the
    recovery consensus's disk half) and point the tracker at the newest
    remaining one and its anchoring base.  Returns the pruned iterations."""
    S = _errors()
    pruned = []
    if not cfg.root.exists():
        return pruned
    with cfg.lock():
        for it in list_iterations(cfg):
            if it > iteration:
                shutil.rmtree(cfg.iter_dir(it), ignore_errors=True)
                pruned.append(it)
        remaining = list_iterations(cfg)
        if not remaining:
            cfg.tracker_path().unlink(missing_ok=True)
            return pruned
        latest = base = max(remaining)
        while True:
            m = read_manifest(cfg, base)
            if m.kind == S.KIND_BASE:
                break
            base = m.base_iteration
        write_tracker(cfg, S.TrackerState(latest, base))
    return pruned


def inspect(cfg: StoreConfig) -> dict:
    """store.py:480-503: the tracker and every checkpoint directory (kind,
    base, record count, tensors.bin size; an unreadable one reports its
    error)."""
    S = _errors()
    tracker = try_read_tracker(cfg)
    rows = []
    for it in list_iterations(cfg):
        try:
            m = read_manifest(cfg, it)
        except S.StoreError as exc:
            rows.append({"iteration": it, "error": str(exc)})
            continue
        rows.append({"iteration": it, "kind": m.kind, "base_iteration": m.base_iteration,
                     "tensors": len(m.tensors),
                     "tensors_bytes": (cfg.iter_dir(it) / "tensors.bin").stat().st_size})
    return {"root": str(cfg.root),
            "tracker": None if tracker is None else {
                "latest_iteration": tracker.latest_iteration,
                "latest_base_iteration": tracker.latest_base_iteration},
            "checkpoints": rows}


def recover_scan(cfg: StoreConfig) -> list:
    """store.py:506-530: after a crash, delete temp debris (.tmp_* dirs, *.tmp
    files) and every checkpoint directory newer than the tracker (never
    committed).  Returns what it did, one line per action."""
    done = []
    if not cfg.root.exists():
        return done
    for p in list(cfg.root.iterdir()):
        if p.name.startswith(".tmp_") or p.suffix == ".tmp":
            if p.is_dir():
                shutil.rmtree(p, ignore_errors=True)
            else:
                p.unlink(missing_ok=True)
            done.append(f"removed temp {p.name}")
    tracker = try_read_tracker(cfg)
    for it in list_iterations(cfg):
        if tracker is None or it > tracker.latest_iteration:
            shutil.rmtree(cfg.iter_dir(it), ignore_errors=True)
            done.append(f"pruned uncommitted iteration {it}")
    return done


def read_manifest(cfg: StoreConfig, iteration: int):
    """store.py:395-410."""
    S = _errors()
    d = cfg.iter_dir(iteration)
    if not d.exists():
        raise S.MissingLinkError(iteration)
    manifest = S.CheckpointManifest.from_bytes((d / "manifest.bin").read_bytes())
    token = (d / "type.txt").read_text().strip()
    if token != manifest.kind:
        raise S.StoreError(f"iteration {iteration}: type.txt says {token!r} but manifest "
                           f"says {manifest.kind!r}")
    if manifest.iteration != iteration:
        raise S.StoreError(f"directory {d.name} holds manifest for iteration "
                           f"{manifest.iteration}")
    return manifest


def load_checkpoint(cfg: StoreConfig, iteration: int | None = None, device=None,
                    to_host: bool = True):
    """store.py:418-474: reconstruct a saved checkpoint.  The chain of
    manifests back to the anchoring base is read from disk, then replayed by
    `decode_chain` on the GPU (model states bit-identical, optimizer states
    dequantized exactly as the reference's dequantize)."""
    S = _errors()
    if iteration is None:
        iteration = read_tracker(cfg).latest_iteration
    chain, it = [], iteration
    while True:
        manifest = read_manifest(cfg, it)
        chain.append(manifest)
        if manifest.kind == S.KIND_BASE:
            break
        it = manifest.base_iteration
    chain.reverse()
    links = [(m, (cfg.iter_dir(m.iteration) / "tensors.bin").read_bytes()) for m in chain]
    return S.decode_chain(links, device=device, to_host=to_host)
