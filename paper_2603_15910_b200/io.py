"""Instance (de)serialization, drop-in for cqksolve/io.py (io.py:1-122),
with binary instances loaded straight into HBM.

Formats (identical bytes to the reference):

* text ``CQK1 <n>`` then d, a, b, l, u (n values each) and r; ``SPX1 <n> <r>``
  then y.  Infinities are spelled ``inf`` / ``-inf``; values use ``%.17g``.
* binary ``CQKB`` / ``SPXB`` magic, n as little-endian u64, then raw
  little-endian float64 in field order (r last for CQK, r first for SPX).

``read_instance(path, device=...)`` reads a binary instance into CUDA tensors
without a pageable detour: the payload is read in chunks (several reader
threads, ``readinto`` releases the GIL) into page-locked staging buffers
whose host-to-device copies overlap the next reads.  The result is
bit-identical to the host read.  Text instances are parsed on the host and
then moved.
"""

import os
import struct
import threading

import numpy as np

from .core import CqkInstance, SimplexInstance, _is_torch

__all__ = ["write_instance", "read_instance", "FormatError"]

_CQK_MAGIC = b"CQKB"
_SPX_MAGIC = b"SPXB"
_CHUNK = 64 << 20  # bytes per staging buffer


class FormatError(ValueError):
    """Unrecognized or corrupt instance file (io.py:26-27)."""


def _fmt(v):
    if v == np.inf:
        return "inf"
    if v == -np.inf:
        return "-inf"
    return f"{v:.17g}"


def _host(a):
    if _is_torch(a):
        return a.detach().to("cpu").numpy()
    return np.asarray(a)


def write_instance(path, inst, binary=False):
    """io.py:38-44.  Device (torch CUDA) instances are copied to the host."""
    if isinstance(inst, CqkInstance):
        _write_cqk(path, inst, binary)
    elif isinstance(inst, SimplexInstance):
        _write_spx(path, inst, binary)
    else:
        raise TypeError(f"cannot serialize {type(inst).__name__}")


def _write_cqk(path, inst, binary):
    arrs = [_host(getattr(inst, f)) for f in ("d", "a", "b", "l", "u")]
    n = int(arrs[0].shape[0])
    if binary:
        with open(path, "wb") as fh:
            fh.write(_CQK_MAGIC)
            fh.write(struct.pack("<Q", n))
            for arr in arrs:
                fh.write(arr.astype("<f8").tobytes())
            fh.write(struct.pack("<d", float(inst.r)))
    else:
        with open(path, "w") as fh:
            fh.write(f"CQK1 {n}\n")
            for arr in arrs:
                fh.write(" ".join(_fmt(v) for v in arr))
                fh.write("\n")
            fh.write(_fmt(float(inst.r)) + "\n")


def _write_spx(path, inst, binary):
    y = _host(inst.y)
    n = int(y.shape[0])
    if binary:
        with open(path, "wb") as fh:
            fh.write(_SPX_MAGIC)
            fh.write(struct.pack("<Q", n))
            fh.write(struct.pack("<d", float(inst.r)))
            fh.write(y.astype("<f8").tobytes())
    else:
        with open(path, "w") as fh:
            fh.write(f"SPX1 {n} {_fmt(float(inst.r))}\n")
            fh.write(" ".join(_fmt(v) for v in y))
            fh.write("\n")


def _load_to_device(path, offset, count, device, workers=4):
    """count float64 values at byte offset of path -> a CUDA tensor, through
    page-locked chunk buffers (reads on `workers` threads, H2D overlapped)."""
    import torch

    out = torch.empty(count, dtype=torch.float64, device=device)
    nbytes = 8 * count
    if nbytes == 0:
        return out
    chunk = min(_CHUNK, nbytes)
    chunk -= chunk % 8
    nchunks = (nbytes + chunk - 1) // chunk
    nbuf = min(2 * workers, nchunks)
    bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(nbuf)]
    done = [torch.cuda.Event() for _ in range(nbuf)]
    stream = torch.cuda.Stream(device=out.device)
    dst = out.view(torch.uint8)
    fd = os.open(path, os.O_RDONLY)
    err = []

    def read_chunk(k, buf):
        want = min(chunk, nbytes - k * chunk)
        view = memoryview(buf.numpy())[:want]
        got = 0
        while got < want:
            n = os.preadv(fd, [view[got:]], offset + k * chunk + got)
            if n <= 0:
                raise FormatError("truncated binary payload")
            got += n
        return want

    try:
        # chunk k uses buffer k % nbuf; reads of the next nbuf chunks run in
        # threads while earlier chunks are in flight to the device
        for k0 in range(0, nchunks, nbuf):
            ks = list(range(k0, min(k0 + nbuf, nchunks)))
            for k in ks:
                done[k % nbuf].synchronize()  # the buffer's previous copy has finished
            sizes = {}

            def work(k):
                try:
                    sizes[k] = read_chunk(k, bufs[k % nbuf])
                except Exception as e:  # surfaced below
                    err.append(e)

            ths = [threading.Thread(target=work, args=(k,)) for k in ks]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if err:
                raise err[0]
            with torch.cuda.stream(stream):
                for k in ks:
                    want = sizes[k]
                    dst[k * chunk:k * chunk + want].copy_(bufs[k % nbuf][:want], non_blocking=True)
                    done[k % nbuf].record(stream)
        stream.synchronize()
    finally:
        os.close(fd)
    return out


def read_instance(path, dtype=np.float64, device=None):
    """Read either format, sniffing text header or binary magic (io.py:80-122).

    device: None -> numpy arrays (the reference's behaviour); a CUDA device
    (e.g. "cuda", 0, torch.device) -> torch tensors resident on it, binary
    payloads streamed straight from the file into HBM.
    """
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(4)
        if head in (_CQK_MAGIC, _SPX_MAGIC):
            raw = fh.read(8)
            if len(raw) != 8:
                raise FormatError("truncated binary header")
            (n,) = struct.unpack("<Q", raw)
            if head == _CQK_MAGIC:
                if size < 12 + 5 * n * 8 + 8:
                    raise FormatError("truncated CQKB payload")
                fh.seek(12 + 5 * n * 8)
                (r,) = struct.unpack("<d", fh.read(8))
                if device is not None:
                    return _device_cqk(path, n, r, dtype, device)
                fh.seek(12)
                body = np.frombuffer(fh.read(5 * n * 8), dtype="<f8")
                d, a, b, l, u = (body[i * n:(i + 1) * n].copy() for i in range(5))
                return CqkInstance(d=d.astype(dtype), a=a.astype(dtype), b=b.astype(dtype),
                                   l=l.astype(dtype), u=u.astype(dtype), r=r)
            if size < 20 + n * 8:
                raise FormatError("truncated SPXB payload")
            (r,) = struct.unpack("<d", fh.read(8))
            if device is not None:
                y = _load_to_device(path, 20, n, _dev(device))
                return SimplexInstance(y=_cast(y, dtype), r=r)
            y = np.frombuffer(fh.read(n * 8), dtype="<f8")
            return SimplexInstance(y=y.copy().astype(dtype), r=r)
    inst = _read_text(path, dtype)
    if device is None:
        return inst
    import torch

    dev = _dev(device)
    if isinstance(inst, CqkInstance):
        return CqkInstance(*[torch.from_numpy(np.ascontiguousarray(getattr(inst, f))).to(dev)
                             for f in ("d", "a", "b", "l", "u")], r=float(inst.r))
    return SimplexInstance(y=torch.from_numpy(inst.y).to(dev), r=float(inst.r))


def _dev(device):
    import torch

    if isinstance(device, int):
        return torch.device("cuda", device)
    return torch.device(device)


def _cast(t, dtype):
    import torch

    if np.dtype(dtype) == np.float32:
        return t.to(torch.float32)
    return t


def _device_cqk(path, n, r, dtype, device):
    dev = _dev(device)
    arrs = [_cast(_load_to_device(path, 12 + i * n * 8, n, dev), dtype) for i in range(5)]
    return CqkInstance(*arrs, r=r)


def _read_text(path, dtype):
    with open(path) as fh:
        tokens = fh.read().split()
    if not tokens:
        raise FormatError("empty instance file")
    kind = tokens[0]
    if kind == "CQK1":
        n = int(tokens[1])
        vals = np.array([float(t) for t in tokens[2:]])
        if vals.size != 5 * n + 1:
            raise FormatError(f"expected {5 * n + 1} values, got {vals.size}")
        d, a, b, l, u = (vals[i * n:(i + 1) * n] for i in range(5))
        return CqkInstance(d=d.astype(dtype), a=a.astype(dtype), b=b.astype(dtype),
                           l=l.astype(dtype), u=u.astype(dtype), r=float(vals[-1]))
    if kind == "SPX1":
        n = int(tokens[1])
        r = float(tokens[2])
        y = np.array([float(t) for t in tokens[3:]])
        if y.size != n:
            raise FormatError(f"expected {n} values, got {y.size}")
        return SimplexInstance(y=y.astype(dtype), r=r)
    raise FormatError(f"unknown instance header {kind!r}")
