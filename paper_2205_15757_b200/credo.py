"""Python front-end over the C-ABI (``include/credo_gpu.h``).

Mirrors the reference's hot-path interface names so callers (and the parity
tests) read like the reference's own code:

================================  ============================================
reference (proj/)                 here
================================  ============================================
crypto::hash                      :meth:`Context.hash_batch`
merkle::leaf_hash                 :meth:`Context.leaf_hash_batch`
merkle::Tree::build(...).root()   :meth:`Context.merkle_roots`
distance::select_quorum           :meth:`Context.select_quorum` /
                                  :meth:`Context.select_quorum_batch`
ModelExecutor::run                :class:`CudaExecutor`
InferenceEngine::execute_batch +  :meth:`ModelGroup.certify`
try_prepare/try_attest digests
================================  ============================================

There is no CPU fallback: constructing a :class:`Context` loads
``libcredo_gpu.so`` and fails loudly when it (or an sm_100a device) is
missing.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CREDO_GPU_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("CREDO_GPU_LIB") or os.path.join(HERE, "libcredo_gpu.so")

CG_OK, CG_EINVAL, CG_ECUDA, CG_ENCCL, CG_EDIGEST, CG_ECODEC, CG_ENOTSUP = range(7)
OP_REQUEST, OP_REQUEST_REJECTED, OP_GROUP = range(3)
EUCLIDEAN, MAX_MINUS_MIN, CHEBYSHEV = 0, 1, 2

u64, u32, dbl, vp = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p


class CredoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(CredoError, ValueError):
    """Where the reference throws std::invalid_argument."""


class DigestMismatch(CredoError):
    pass


class CodecError(CredoError, ValueError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.cg_last_error.restype = C.c_char_p
        L.cg_last_error.argtypes = [vp]
        L.cg_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.cg_ctx_destroy.argtypes = [vp]
        L.cg_ctx_set_stream.argtypes = [vp, vp]
        L.cg_ctx_stream.restype = vp
        L.cg_ctx_stream.argtypes = [vp]
        L.cg_ctx_synchronize.argtypes = [vp]
        L.cg_ctx_launch_count.restype = u64
        L.cg_ctx_launch_count.argtypes = [vp]
        L.cg_model_free.argtypes = [vp]
        L.cg_group_free.argtypes = [vp]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _unpack_paths(sib, sides, lens, count):
    return [[(sib[t, k].tobytes(), int(sides[t, k])) for k in range(int(lens[t]))]
            for t in range(count)]


def _pack_paths(paths):
    c = max(len(paths), 1)
    sib = np.zeros((c, 64, 32), np.uint8)
    sides = np.zeros((c, 64), np.uint8)
    lens = np.zeros(c, np.uint32)
    for t, p in enumerate(paths):
        lens[t] = len(p)
        for k, (s, d) in enumerate(p):
            sib[t, k] = np.frombuffer(s, np.uint8)
            sides[t, k] = d
    return sib, sides, lens


# ---------------------------------------------------------------- context
class Context:
    """One context per process/GPU (cg_ctx)."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = vp()
        rc = self.L.cg_ctx_create(device, C.byref(h))
        if rc != CG_OK:
            raise CredoError(rc, f"cg_ctx_create(device={device}) failed "
                                 "(needs an sm_100a B200)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.cg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc == CG_OK:
            return
        msg = self.L.cg_last_error(self.h).decode(errors="replace")
        cls = {CG_EINVAL: InvalidArgument, CG_EDIGEST: DigestMismatch,
               CG_ECODEC: CodecError}.get(rc, CredoError)
        raise cls(rc, msg)

    def set_stream(self, stream_ptr: int):
        self._check(self.L.cg_ctx_set_stream(self.h, vp(stream_ptr)))

    @property
    def stream(self) -> int:
        return self.L.cg_ctx_stream(self.h) or 0

    def synchronize(self):
        self._check(self.L.cg_ctx_synchronize(self.h))

    def join(self):
        """The context stream waits for all certification tails so far."""
        self._check(self.L.cg_ctx_join(self.h))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        rc = lib().cg_nccl_unique_id(buf)
        if rc != CG_OK:
            raise CredoError(rc, "ncclGetUniqueId failed")
        return buf.raw

    def init_nccl(self, uid: bytes, nranks: int, rank: int):
        """One rank per GPU; uid from rank 0's nccl_unique_id()."""
        assert len(uid) == 128
        self._check(self.L.cg_ctx_init_nccl(self.h, uid, nranks, rank))

    def launch_count(self) -> int:
        return int(self.L.cg_ctx_launch_count(self.h))

    # -- digests ----------------------------------------------------------
    def _msgs(self, msgs: Sequence[bytes]):
        lens = np.array([len(m) for m in msgs], np.uint64)
        offs = np.zeros(len(msgs), np.uint64)
        if len(msgs) > 1:
            offs[1:] = np.cumsum(lens[:-1])
        return b"".join(msgs), offs, lens

    def hash_batch(self, msgs: Sequence[bytes]) -> list[bytes]:
        """crypto::hash over each message (crypto.cpp:22-27)."""
        buf, offs, lens = self._msgs(msgs)
        out = C.create_string_buffer(32 * max(1, len(msgs)))
        self._check(self.L.cg_sha256_batch(self.h, buf, _p(offs), _p(lens),
                                           u64(len(msgs)), out))
        return [out.raw[32 * i:32 * i + 32] for i in range(len(msgs))]

    def hash(self, data: bytes) -> bytes:
        return self.hash_batch([data])[0]

    def leaf_hash_batch(self, leaves: Sequence[bytes]) -> list[bytes]:
        """merkle::leaf_hash = H(0x00 || leaf) (merkle.cpp:22-25)."""
        buf, offs, lens = self._msgs(leaves)
        out = C.create_string_buffer(32 * max(1, len(leaves)))
        self._check(self.L.cg_leaf_hash_batch(self.h, buf, _p(offs), _p(lens),
                                              u64(len(leaves)), out))
        return [out.raw[32 * i:32 * i + 32] for i in range(len(leaves))]

    def merkle_roots(self, trees: Sequence[Sequence[bytes]]) -> list[bytes]:
        """Tree::build(...).root() over precomputed leaf hashes per tree."""
        n = np.array([len(t) for t in trees], np.uint64)
        buf = b"".join(b"".join(t) for t in trees)
        out = C.create_string_buffer(32 * max(1, len(trees)))
        self._check(self.L.cg_merkle_root_batch(self.h, buf, _p(n),
                                                u64(len(trees)), out))
        return [out.raw[32 * i:32 * i + 32] for i in range(len(trees))]

    def auth_paths(self, leaf_hashes: Sequence[bytes], indices):
        """Tree::build over the leaf hashes; auth_path(i) for each index as
        [(sibling, side)] (side 0 = left, 1 = right), plus the root."""
        n = len(leaf_hashes)
        idx = np.ascontiguousarray(indices, np.uint64)
        c = len(idx)
        sib = np.zeros((max(c, 1), 64, 32), np.uint8)
        sides = np.zeros((max(c, 1), 64), np.uint8)
        lens = np.zeros(max(c, 1), np.uint32)
        root = np.zeros(32, np.uint8)
        self._check(self.L.cg_merkle_auth_paths(self.h, b"".join(leaf_hashes) or b"\0", u64(n),
                                                _p(idx), u32(c), _p(sib), _p(sides), _p(lens),
                                                _p(root)))
        return _unpack_paths(sib, sides, lens, c), root.tobytes()

    def path_roots(self, leaf_hashes: Sequence[bytes], paths) -> list[bytes]:
        """merkle::get_merkle_root for each (leaf hash, path)."""
        sib, sides, lens = _pack_paths(paths)
        out = np.zeros((max(len(paths), 1), 32), np.uint8)
        self._check(self.L.cg_merkle_path_roots(self.h, b"".join(leaf_hashes) or b"\0",
                                                _p(sib), _p(sides), _p(lens), u32(len(paths)),
                                                _p(out)))
        return [out[i].tobytes() for i in range(len(paths))]

    # -- agreement ----------------------------------------------------------
    def select_quorum_batch(self, outs: np.ndarray, n: int, f: int,
                            metric: int, eps, present=None, with_label=True):
        """outs: (R, n, v). Returns dict of arrays; raises InvalidArgument
        where distance::select_quorum would throw (status marks which)."""
        outs = np.ascontiguousarray(outs, np.float64)
        R, n_, v = outs.shape
        assert n_ == n
        eps = np.ascontiguousarray(np.broadcast_to(np.asarray(eps, np.float64), (R,)))
        pres = None if present is None else np.ascontiguousarray(present, np.uint32)
        sel = np.zeros(R, np.uint32)
        diam = np.zeros(R, np.float64)
        sat = np.zeros(R, np.uint8)
        status = np.zeros(R, np.int8)
        label = np.zeros(R, np.int64) if with_label else None
        rc = self.L.cg_select_quorum_batch(self.h, _p(outs), _p(pres), _p(eps),
                                           u32(R), u32(n), u32(f), u32(v),
                                           u32(metric), _p(sel), _p(diam),
                                           _p(sat), _p(status), _p(label))
        res = dict(selected=sel, diameter=diam, satisfied=sat.astype(bool),
                   status=status, label=label)
        if rc != CG_OK:
            err = InvalidArgument if rc == CG_EINVAL else CredoError
            e = err(rc, self.L.cg_last_error(self.h).decode())
            e.result = res
            raise e
        return res

    def agree_device(self, outs_ptr: int, ps: int, rs: int, eps_ptr: int, R: int, n: int,
                     f: int, v: int, metric: int, sel_ptr: int, diam_ptr: int, sat_ptr: int,
                     status_ptr: int, label_ptr: int = 0, req_ids_ptr: int = 0,
                     version: int = 0, digest_ptr: int = 0):
        """cg_agree_device: device pointers (e.g. torch tensors' data_ptr()),
        enqueued on this context's stream without a host sync."""
        vp_ = lambda x: vp(x) if x else None  # noqa: E731
        L = self.L
        L.cg_agree_device.argtypes = [vp, vp, u64, u64, vp, u32, u32, u32, u32, u32, vp, u64,
                                      vp, vp, vp, vp, vp, vp]
        self._check(L.cg_agree_device(self.h, vp_(outs_ptr), ps, rs, vp_(eps_ptr), R, n, f, v,
                                      metric, vp_(req_ids_ptr), version, vp_(sel_ptr),
                                      vp_(diam_ptr), vp_(sat_ptr), vp_(status_ptr),
                                      vp_(label_ptr), vp_(digest_ptr)))

    def label_digests(self, req_ids: np.ndarray, labels: np.ndarray, version: int) -> np.ndarray:
        """SHA-256(0x4C || id || u64be version || u64be label) per request."""
        ids = np.ascontiguousarray(req_ids, np.uint8).reshape(-1, 32)
        lab = np.ascontiguousarray(labels, np.int64)
        out = np.zeros((len(lab), 32), np.uint8)
        self._check(self.L.cg_label_digest_batch(self.h, _p(ids), _p(lab), u32(len(lab)),
                                                 u64(version), _p(out)))
        return out

    def synth_outputs(self, seed: int, R: int, n: int, v: int, eps: float, shift_frac: float,
                      outs_ptr: int, ids_ptr: int = 0):
        """C5 synthetic per-replica outputs generated on the device."""
        L = self.L
        L.cg_synth_outputs.argtypes = [vp, u64, u32, u32, u32, dbl, dbl, vp, vp]
        self._check(L.cg_synth_outputs(self.h, seed, R, n, v, eps, shift_frac, vp(outs_ptr),
                                       vp(ids_ptr) if ids_ptr else None))

    def request_digests(self, batch: "RequestBatch", group_id: bytes):
        """verify_request's device part for a batch: (signing digests
        SHA-256(0x01 || body), canonical ids, status 0 ok / 1 empty nonce /
        2 empty input / 3 bad epsilon / 4 id mismatch)."""
        cb, keep, B = ModelGroup._cbatch(batch)
        sig = np.zeros((B, 32), np.uint8)
        ids = np.zeros((B, 32), np.uint8)
        st = np.zeros(B, np.int8)
        self._check(self.L.cg_request_digests(self.h, C.byref(cb), group_id, u64(len(group_id)),
                                              _p(sig), _p(ids), _p(st)))
        return sig, ids, st

    def cert_leaf_hashes(self, batch: "RequestBatch", group_id: bytes, req_index, want,
                         results):
        """cg_cert_leaf_hashes: per entry m, leaf_hash of result_leaf (want
        bit 1), single_attest_leaf (bit 2) of (request req_index[m],
        results[m] = InferenceResult::encode bytes) or missing_result_leaf
        (bit 4) -- the leaves verify_cert / assemble_response re-hash.
        Returns (leaf52, leaf53, leaf4d), each M x 32 (zeros where not wanted)."""
        cb, keep, B = ModelGroup._cbatch(batch)
        M = len(req_index)
        ridx = np.ascontiguousarray(req_index, np.uint32)
        w = np.ascontiguousarray(want, np.uint8)
        lens = np.array([len(r) for r in results], np.uint64)
        enc = np.frombuffer(b"".join(results) or b"\0", np.uint8)
        out = [np.zeros((M, 32), np.uint8) for _ in range(3)]
        self._check(self.L.cg_cert_leaf_hashes(
            self.h, C.byref(cb), group_id, u64(len(group_id)), C.c_uint32(M), _p(ridx), _p(w),
            _p(enc), _p(lens), _p(out[0]), _p(out[1]), _p(out[2])))
        return tuple(out)

    def select_quorum(self, results: dict, n: int, f: int, metric: int,
                      epsilon: float):
        """distance::select_quorum(map<node, vector<double>>, n, f, m, eps)."""
        if not results:
            raise InvalidArgument(CG_EINVAL, "select_quorum: no results")
        v = len(next(iter(results.values())))
        outs = np.zeros((1, n, max(v, 1)), np.float64)
        present = 0
        for node, vec in results.items():
            if node >= n or node >= 32:
                raise InvalidArgument(CG_EINVAL, "node index out of range")
            if len(vec) != v:
                raise InvalidArgument(CG_EINVAL, "result dimensionality mismatch")
            outs[0, node, :] = vec
            present |= 1 << node
        r = self.select_quorum_batch(outs, n, f, metric, [epsilon],
                                     present=[present], with_label=False)
        sel = int(r["selected"][0])
        return AgreementOutcome(
            selected={i for i in range(32) if sel >> i & 1},
            diameter=float(r["diameter"][0]), satisfied=bool(r["satisfied"][0]))


class _COpsBatch(C.Structure):
    _fields_ = [("requests", vp), ("group_id", C.c_char_p), ("group_id_len", u64),
                ("version", u64), ("versions", vp), ("statuses", vp), ("reasons", C.c_char_p),
                ("reason_lens", vp)]


def host_sha256(data: bytes) -> bytes:
    """SHA-256 on the host (SHA-NI when present): the model-file check."""
    out = C.create_string_buffer(32)
    rc = lib().cg_host_sha256(data, u64(len(data)), out)
    if rc != CG_OK:
        raise CredoError(rc, "cg_host_sha256 failed")
    return out.raw


def hash_ops_batches(batches: Sequence["RequestBatch"], group_id: bytes, versions,
                     statuses=None, reasons=None, threads: int = 1) -> list[bytes]:
    """hash_ops (messages.cpp:197-202) of one PRE-PREPARE op list per batch
    (every op an inference request), host SHA-NI, one op list per thread.
    versions[i]: an int or a per-request sequence; statuses / reasons the
    same (None: ok / "")."""
    keep, arr = [], (_COpsBatch * max(1, len(batches)))()
    for i, b in enumerate(batches):
        cb, k, B = ModelGroup._cbatch(b)
        keep += [cb, k]
        v = versions[i]
        vs = None if np.isscalar(v) else np.ascontiguousarray(v, np.uint64)
        st = None if statuses is None else np.ascontiguousarray(statuses[i], np.uint8)
        rs = rl = None
        if reasons is not None:
            enc = [r.encode() for r in reasons[i]]
            rs = b"".join(enc) or b"\0"
            rl = np.array([len(r) for r in enc], np.uint64)
        keep += [vs, st, rs, rl]
        arr[i] = _COpsBatch(C.cast(C.pointer(cb), vp), group_id, len(group_id),
                            int(v) if vs is None else 0, _p(vs), _p(st), rs, _p(rl))
    out = C.create_string_buffer(32 * max(1, len(batches)))
    rc = lib().cg_hash_ops_batches(arr, u32(len(batches)), C.c_int(threads), out)
    if rc != CG_OK:
        raise CredoError(rc, "cg_hash_ops_batches: bad arguments")
    return [out.raw[32 * i:32 * i + 32] for i in range(len(batches))]


class _CRequest(C.Structure):
    _fields_ = [("request_id", vp), ("group_id", C.c_char_p), ("group_id_len", u64),
                ("input", vp), ("input_dim", u64), ("has_eps", C.c_int), ("eps", dbl),
                ("client_pub", vp), ("nonce", C.c_char_p), ("nonce_len", u64),
                ("client_sig", vp)]


class _CReady(C.Structure):
    _fields_ = [("group", vp), ("version", u64), ("ticket", u64), ("B", u32)]


SUBMIT_OK, SUBMIT_INVALID, SUBMIT_UNKNOWN_GROUP, SUBMIT_RETIRED = range(4)
GROUP_DEFINED, GROUP_ACTIVE, GROUP_RETIRED = range(3)


class InferenceEngine:
    """The batch former (InferenceEngine::submit / flush_due / flush_version /
    flush_all / next_flush_deadline, engine.cpp:166-267) over GPU groups:
    per live (group, version) FIFO with seen-dedup, batches of
    exec_batch_max or flushed partial ones, packed into pinned staging as
    requests arrive and ingested into the group; ready() returns
    (group, version, ticket, B) in release order for certify_ticket."""

    def __init__(self, ctx: Context, exec_batch_max: int, flush_interval_us: int,
                 pack_threads: int = 1):
        self.ctx = ctx
        h = vp()
        ctx._check(ctx.L.cg_engine_create(ctx.h, u64(exec_batch_max), u64(flush_interval_us),
                                          C.c_int(pack_threads), C.byref(h)))
        self.h = h
        self._groups = {}

    def free(self):
        if self.h:
            self.ctx.L.cg_engine_free(self.h)
            self.h = None

    def load_group(self, group: "ModelGroup", status: int = GROUP_ACTIVE):
        self.ctx._check(self.ctx.L.cg_engine_load_group(self.h, group.h, C.c_int(status)))
        self._groups[group.h.value] = group

    def set_status(self, group_id: bytes, version: int, status: int):
        self.ctx._check(self.ctx.L.cg_engine_set_status(self.h, group_id, u64(len(group_id)),
                                                        u64(version), C.c_int(status)))

    def submit(self, batch: RequestBatch, now_us: int, group_id: bytes = b"group-0"):
        """Submits the batch's requests in order; returns the per-request
        SubmitOutcome error codes (SUBMIT_*)."""
        return self.submit_prepared(self.prepare(batch, group_id), now_us)

    def prepare(self, batch: RequestBatch, group_id: bytes = b"group-0"):
        """The cg_request array of a batch (pointers into its arrays; keep
        the batch alive), reusable across submit_prepared calls."""
        n = len(batch.nonces)
        rows = batch.inputs if isinstance(batch.inputs, (list, tuple)) else \
            np.ascontiguousarray(batch.inputs, np.float64)
        rows = [np.ascontiguousarray(rows[k], np.float64).ravel() for k in range(n)]
        ids = np.ascontiguousarray(batch.request_ids, np.uint8)
        pubs = np.ascontiguousarray(batch.client_pubs, np.uint8)
        sigs = np.ascontiguousarray(batch.client_sigs, np.uint8)
        arr = (_CRequest * max(n, 1))()
        for k in range(n):
            e = None if batch.eps is None else batch.eps[k]
            arr[k] = _CRequest(ids[k].ctypes.data, group_id, len(group_id), rows[k].ctypes.data,
                               len(rows[k]), int(e is not None), e or 0.0, pubs[k].ctypes.data,
                               batch.nonces[k], len(batch.nonces[k]), sigs[k].ctypes.data)
        return (arr, n, [rows, ids, pubs, sigs, batch])

    def submit_prepared(self, prepared, now_us: int):
        arr, n, _keep = prepared
        err = np.zeros(max(n, 1), np.int32)
        self.ctx._check(self.ctx.L.cg_engine_submit(self.h, arr, u32(n), u64(now_us), _p(err)))
        return err[:n].tolist()

    def flush_due(self, now_us: int):
        self.ctx._check(self.ctx.L.cg_engine_flush_due(self.h, u64(now_us)))

    def flush_version(self, group_id: bytes, version: int):
        self.ctx._check(self.ctx.L.cg_engine_flush_version(self.h, group_id, u64(len(group_id)),
                                                           u64(version)))

    def flush_all(self):
        self.ctx._check(self.ctx.L.cg_engine_flush_all(self.h))

    def next_flush_deadline(self) -> Optional[int]:
        d, has = u64(), C.c_int()
        self.ctx._check(self.ctx.L.cg_engine_next_flush_deadline(self.h, C.byref(d), C.byref(has)))
        return d.value if has.value else None

    def ready(self):
        """[(ModelGroup, version, ticket, B)] released since the last call."""
        out = []
        while True:
            buf = (_CReady * 64)()
            n = u32()
            self.ctx._check(self.ctx.L.cg_engine_ready(self.h, buf, u32(64), C.byref(n)))
            for i in range(n.value):
                r = buf[i]
                out.append((self._groups[r.group], r.version, r.ticket, r.B))
            if n.value < 64:
                return out

    def pending(self):
        q, w = u64(), u64()
        self.ctx._check(self.ctx.L.cg_engine_pending(self.h, C.byref(q), C.byref(w)))
        return q.value, w.value


@dataclass
class AgreementOutcome:
    """distance::AgreementOutcome (distance.hpp:55-59)."""
    selected: set = field(default_factory=set)
    diameter: float = 0.0
    satisfied: bool = False


# ------------------------------------------------------------------ models
class Model:
    def __init__(self, ctx: Context, h, digest: bytes, arch: str = "linear"):
        self.ctx, self.h, self.digest, self.arch = ctx, h, digest, arch
        u, v = u64(), u64()
        ctx.L.cg_model_dims(h, C.byref(u), C.byref(v))
        self.input_dim, self.output_dim = u.value, v.value

    @classmethod
    def load_linear(cls, ctx: Context, file: bytes, digest: bytes) -> "Model":
        """LinearToyModel::from_file_bytes + the load_group digest check."""
        h = vp()
        ctx._check(ctx.L.cg_model_load_linear(ctx.h, file, u64(len(file)),
                                              digest, C.byref(h)))
        return cls(ctx, h, digest)

    @classmethod
    def load_cnn(cls, ctx: Context, file: bytes, digest: bytes) -> "Model":
        h = vp()
        ctx._check(ctx.L.cg_model_load_cnn(ctx.h, file, u64(len(file)),
                                           digest, C.byref(h)))
        # canonical header: str magic | str arch | ...
        ml = int.from_bytes(file[0:4], "big")
        al = int.from_bytes(file[4 + ml:8 + ml], "big")
        return cls(ctx, h, digest, file[8 + ml:8 + ml + al].decode())

    def free(self):
        if self.h:
            self.ctx.L.cg_model_free(self.h)
            self.h = None


class CudaExecutor:
    """ModelExecutor::run (model.hpp:48-50): one output per input, in order."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def run(self, model: Model, inputs) -> np.ndarray:
        x = np.ascontiguousarray(inputs, np.float64)
        if x.ndim == 1:
            x = x[None]
        B, u = x.shape
        y = np.zeros((B, model.output_dim), np.float64)
        self.ctx._check(self.ctx.L.cg_exec_run(self.ctx.h, model.h, _p(x),
                                               u64(B), u64(u), _p(y),
                                               u64(model.output_dim)))
        return y


class PerturbingExecutor:
    """PerturbingExecutor(inner, node_index, magnitude) (model.hpp:60-79,
    model.cpp:75-105) around the CUDA executor: each lane gets the node's
    deterministic offset from SHA-256(node || model digest || input || lane),
    computed on the GPU (midstate chain jobs + one thread per lane)."""

    def __init__(self, ctx: Context, node_index: int, magnitude: float):
        if not (magnitude >= 0.0):
            raise ValueError("negative magnitude")
        self.ctx, self.node_index, self.magnitude = ctx, node_index, magnitude

    def run(self, model: Model, inputs) -> np.ndarray:
        x = np.ascontiguousarray(inputs, np.float64)
        if x.ndim == 1:
            x = x[None]
        B, u = x.shape
        y = np.zeros((B, model.output_dim), np.float64)
        self.ctx._check(self.ctx.L.cg_exec_run_perturbed(
            self.ctx.h, model.h, _p(x), u64(B), u64(u), _p(y),
            u64(model.output_dim), u64(self.node_index), C.c_double(self.magnitude)))
        return y


# ------------------------------------------------------------ request batch
@dataclass
class RequestBatch:
    """ExecutionBatch (engine.hpp:29-34) in struct-of-arrays form."""
    request_ids: np.ndarray          # (B, 32) uint8
    inputs: object                   # (B, u) float64 ndarray, or device ptr
    client_pubs: np.ndarray          # (B, 32) uint8
    nonces: list                     # B × bytes
    client_sigs: np.ndarray          # (B, 64) uint8
    eps: Optional[list] = None       # B × (float | None)
    u: Optional[int] = None
    B: Optional[int] = None
    # optional PRE-PREPARE op-list structure (cg_request_batch.op_kinds):
    # per op OP_REQUEST / OP_REQUEST_REJECTED / OP_GROUP, the group ops'
    # OpEntry encodings and the rejected ops' FailureRecord encodings
    op_kinds: Optional[list] = None
    op_entries: Optional[list] = None    # B x bytes (b"" for requests)
    fail_records: Optional[list] = None  # B x bytes (b"" when not rejected)

    @classmethod
    def from_encoded(cls, encs: Sequence[bytes]) -> "RequestBatch":
        """Decode InferenceRequest::encode bytes (domain.cpp:153-175)."""
        ids, inputs, pubs, nonces, sigs, eps = [], [], [], [], [], []
        for buf in encs:
            off = 32
            ids.append(np.frombuffer(buf[:32], np.uint8))
            gl = struct.unpack(">I", buf[off:off + 4])[0]; off += 4 + gl
            n = struct.unpack(">I", buf[off:off + 4])[0]; off += 4
            inputs.append(np.frombuffer(buf[off:off + 8 * n], ">f8").astype(np.float64)); off += 8 * n
            has = buf[off]; off += 1
            if has:
                eps.append(struct.unpack(">d", buf[off:off + 8])[0]); off += 8
            else:
                eps.append(None)
            pubs.append(np.frombuffer(buf[off:off + 32], np.uint8)); off += 32
            nl = struct.unpack(">I", buf[off:off + 4])[0]; off += 4
            nonces.append(bytes(buf[off:off + nl])); off += nl
            sigs.append(np.frombuffer(buf[off:off + 64], np.uint8)); off += 64
            if off != len(buf):
                raise CodecError(CG_ECODEC, "trailing bytes after value")
        ragged = len({len(x) for x in inputs}) > 1  # misfit requests: keep rows
        return cls(np.stack(ids), inputs if ragged else np.stack(inputs), np.stack(pubs), nonces,
                   np.stack(sigs), eps if any(e is not None for e in eps) else None)


class _CReqBatch(C.Structure):
    _fields_ = [("B", u32), ("u", u64), ("request_ids", vp), ("inputs", vp),
                ("inputs_on_device", C.c_int), ("has_eps", vp), ("eps", vp),
                ("client_pubs", vp), ("nonces", vp), ("nonce_lens", vp),
                ("client_sigs", vp), ("input_dims", vp), ("misfit_inputs", vp),
                ("op_kinds", vp), ("op_entries", vp), ("op_entry_lens", vp),
                ("fail_records", vp), ("fail_record_lens", vp)]


class _COut(C.Structure):
    _fields_ = [(n, vp) for n in (
        "selected", "diameter", "satisfied", "label", "r_roots", "a_root",
        "manifest_len", "manifest_kind", "manifest_node", "manifest_op",
        "leaf_hashes", "a_leaf_hashes", "outputs", "topk_idx", "topk_val")]


class ModelGroup:
    """A model group's replica set on this GPU: models[p] answers as node p."""

    def __init__(self, ctx: Context, models: Sequence[Model], f: int,
                 metric: int, default_eps: float, group_id: bytes,
                 version: int, max_batch: int, topk: int = 5):
        self.ctx, self.models = ctx, list(models)
        self.N, self.f, self.topk = len(models), f, topk
        self.v = models[0].output_dim
        self.u = models[0].input_dim
        self.group_id, self.version = group_id, version
        self.default_eps = default_eps
        arr = (vp * len(models))(*[m.h for m in models])
        h = vp()
        ctx._check(ctx.L.cg_group_create(ctx.h, arr, u32(len(models)), u32(f),
                                         u32(metric), dbl(default_eps),
                                         group_id, u64(len(group_id)),
                                         u64(version), u32(max_batch),
                                         u32(topk), C.byref(h)))
        self.h = h
        self._keep = None

    ring = 24  # CG_INGEST_RING: batches in flight per group

    @classmethod
    def create_dist(cls, ctx: Context, my_model, digests: Sequence[bytes],
                    f: int, metric: int, default_eps: float, group_id: bytes,
                    version: int, max_batch: int, topk: int = 5) -> "ModelGroup":
        """Replica-parallel group: this rank (ctx.init_nccl) serves provider
        `rank` (my_model), or with a list of k models providers
        [rank k, (rank + 1) k); digests lists every provider's."""
        mine = list(my_model) if isinstance(my_model, (list, tuple)) else [my_model]
        self = cls.__new__(cls)
        self.ctx, self.models = ctx, mine
        self.N, self.f, self.topk = len(digests), f, topk
        self.v, self.u = mine[0].output_dim, mine[0].input_dim
        self.group_id, self.version = group_id, version
        self.default_eps = default_eps
        h = vp()
        arr = (vp * len(mine))(*[m.h for m in mine])
        ctx._check(ctx.L.cg_group_create_dist_multi(ctx.h, arr, u32(len(mine)),
                                                    b"".join(digests), u32(f), u32(metric),
                                                    dbl(default_eps), group_id,
                                                    u64(len(group_id)), u64(version),
                                                    u32(max_batch), u32(topk), C.byref(h)))
        self.h = h
        self._keep = None
        return self

    def auth_paths(self, tree: int, indices, ticket: Optional[int] = None):
        """Paths in provider `tree`'s result tree (tree < N) or the
        attestation tree (tree == N) of the last certified batch (or of the
        certified `ticket`)."""
        idx = np.ascontiguousarray(indices, np.uint64)
        c = len(idx)
        sib = np.zeros((max(c, 1), 64, 32), np.uint8)
        sides = np.zeros((max(c, 1), 64), np.uint8)
        lens = np.zeros(max(c, 1), np.uint32)
        L = self.ctx.L
        if ticket is None:
            rc = L.cg_group_auth_paths(self.h, u32(tree), _p(idx), u32(c), _p(sib), _p(sides),
                                       _p(lens))
        else:
            rc = L.cg_group_auth_paths_ticket(self.h, u64(ticket), u32(tree), _p(idx), u32(c),
                                              _p(sib), _p(sides), _p(lens))
        self.ctx._check(rc)
        return _unpack_paths(sib, sides, lens, c)

    def free(self):
        if self.h:
            self.ctx.L.cg_group_free(self.h)
            self.h = None

    @staticmethod
    def _cbatch(b: RequestBatch, group_u: Optional[int] = None):
        """RequestBatch -> cg_request_batch. b.inputs: (B, u) array, a device
        pointer, or (ragged) a list of 1-D arrays: rows whose length is not
        group_u are misfits (execute_batch skips them)."""
        dims = mis = None
        if isinstance(b.inputs, (list, tuple)):
            assert group_u is not None
            rows = [np.ascontiguousarray(r, np.float64).ravel() for r in b.inputs]
            x = np.zeros((len(rows), group_u), np.float64)
            dims = np.array([len(r) for r in rows], np.uint64)
            mis = (vp * len(rows))(*[r.ctypes.data if len(r) else None for r in rows])
            for k, r in enumerate(rows):
                if len(r) == group_u:
                    x[k] = r
            import dataclasses
            b = dataclasses.replace(b, inputs=x)
            misfit_keep = (rows, dims, mis)
        else:
            misfit_keep = None
        on_dev = not isinstance(b.inputs, np.ndarray)
        if on_dev:
            inputs_ptr, B, u = int(b.inputs), int(b.B), int(b.u)
        else:
            x = np.ascontiguousarray(b.inputs, np.float64)
            inputs_ptr, (B, u) = x.ctypes.data, x.shape
        ids = np.ascontiguousarray(b.request_ids, np.uint8)
        pubs = np.ascontiguousarray(b.client_pubs, np.uint8)
        sigs = np.ascontiguousarray(b.client_sigs, np.uint8)
        nl = np.array([len(n) for n in b.nonces], np.uint64)
        nb = np.frombuffer(b"".join(b.nonces) or b"\0", np.uint8).copy()
        has = eps = None
        if b.eps is not None:
            has = np.array([e is not None for e in b.eps], np.uint8)
            eps = np.array([e or 0.0 for e in b.eps], np.float64)
        kinds = ents = el = recs = rl = None
        if b.op_kinds is not None:
            kinds = np.ascontiguousarray(b.op_kinds, np.uint8)
            e = b.op_entries or [b""] * B
            r = b.fail_records or [b""] * B
            el = np.array([len(x) for x in e], np.uint64)
            rl = np.array([len(x) for x in r], np.uint64)
            ents = np.frombuffer(b"".join(e) or b"\0", np.uint8).copy()
            recs = np.frombuffer(b"".join(r) or b"\0", np.uint8).copy()
        keep = [ids, pubs, sigs, nl, nb, has, eps,
                None if on_dev else x, misfit_keep, kinds, ents, el, recs, rl]
        cb = _CReqBatch(B, u, ids.ctypes.data, inputs_ptr, int(on_dev),
                        None if has is None else has.ctypes.data,
                        None if eps is None else eps.ctypes.data,
                        pubs.ctypes.data, nb.ctypes.data, nl.ctypes.data,
                        sigs.ctypes.data,
                        None if dims is None else dims.ctypes.data,
                        None if mis is None else C.cast(mis, vp),
                        *[None if z is None else z.ctypes.data for z in (kinds, ents, el, recs, rl)])
        return cb, keep, B

    def encode_results(self, provider: int, ticket: Optional[int] = None) -> bytes:
        """encode_results (messages.cpp:48-50) of one provider's results for
        the last certified batch (or the certified `ticket`): the PREPARE /
        PRE-PREPARE result payload."""
        L, n = self.ctx.L, u64()
        if ticket is None:
            call = lambda buf, cap: L.cg_group_encode_results(  # noqa: E731
                self.h, C.c_uint32(provider), buf, u64(cap), C.byref(n))
        else:
            call = lambda buf, cap: L.cg_group_encode_results_ticket(  # noqa: E731
                self.h, u64(ticket), C.c_uint32(provider), buf, u64(cap), C.byref(n))
        self.ctx._check(call(None, 0))
        buf = C.create_string_buffer(max(n.value, 1))
        self.ctx._check(call(buf, n.value))
        return buf.raw[:n.value]

    def set_fault(self, provider: int, offset: float, fraction: float = 1.0):
        """OffsetExecutor(offset) around provider `provider` (the
        corrupt_result fault, harness.cpp:167-186) for the requests whose
        first id byte is < round(256 * fraction)."""
        self.ctx._check(self.ctx.L.cg_group_set_fault(self.h, C.c_uint32(provider),
                                                      C.c_double(offset), C.c_double(fraction)))

    def set_perturbation(self, magnitude: float):
        """PerturbingExecutor around every replica (harness.cpp:255-258)."""
        self.ctx._check(self.ctx.L.cg_group_set_perturbation(self.h, C.c_double(magnitude)))

    def certify(self, batch: RequestBatch, want_outputs: bool = False,
                want_leaves: bool = False, sync: bool = True):
        """One ExecutionBatch through the hot path. sync=False only enqueues
        (results stay on the device; call :meth:`fetch`)."""
        cb, keep, B = self._cbatch(batch, self.u)
        self._keep = keep
        if not sync:
            self.ctx._check(self.ctx.L.cg_certify_batch(self.h, C.byref(cb), None))
            self._lastB = B
            return None
        self._lastB = B
        return self.fetch(want_outputs, want_leaves, _enqueue=(cb,))

    def ingest(self, batch: RequestBatch) -> int:
        """InferenceEngine::submit's hot part: frame, upload and start the
        request-midstate chains. Returns a ticket for :meth:`certify_ticket`."""
        cb, keep, B = self._cbatch(batch, self.u)
        t = C.c_uint64()
        self.ctx._check(self.ctx.L.cg_ingest_batch(self.h, C.byref(cb), C.byref(t)))
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[t.value] = (keep, B)   # host inputs may still be in flight
        return t.value

    def certify_ticket(self, ticket: int, sync: bool = True, want_outputs=False,
                       want_leaves=False, B: Optional[int] = None):
        """B: the batch size, for tickets ingested by an InferenceEngine."""
        self._inflight = getattr(self, "_inflight", {})
        keep, B = self._inflight.pop(ticket, (None, B))
        self._lastB = B
        self._doneB = getattr(self, "_doneB", {})
        self._doneB[ticket] = B
        if len(self._doneB) > 64:
            self._doneB.pop(next(iter(self._doneB)))
        if not sync:
            self.ctx._check(self.ctx.L.cg_certify_ticket(self.h, C.c_uint64(ticket), None))
            self._keep = keep
            return None
        return self.fetch(want_outputs, want_leaves, _ticket=ticket)

    def certify_outputs(self, batch: RequestBatch, outputs: np.ndarray,
                        want_leaves: bool = False):
        """Agreement + digests over precomputed (N, B, v) replica outputs
        (C5 sweep / fault injection: a corrupt replica is a shifted row)."""
        cb, keep, B = self._cbatch(batch, self.u)
        o = np.ascontiguousarray(outputs, np.float64)
        assert o.shape == (self.N, B, self.v)
        self._keep = keep + [o]
        self._lastB = B
        return self.fetch(False, want_leaves, _enqueue=(cb,), _outputs=o)

    def certify_empty_slot(self, view: int, seq: int):
        """An empty filler slot: noop_leaf R trees, N whole-batch A leaves."""
        N = self.N
        r = dict(r_roots=np.zeros((N, 32), np.uint8), a_root=np.zeros(32, np.uint8),
                 manifest_len=np.zeros(1, np.uint64), manifest_kind=np.zeros(N, np.uint8),
                 manifest_node=np.zeros(N, np.uint32), manifest_op=np.zeros(N, np.uint32),
                 a_leaf_hashes=np.zeros((N, 32), np.uint8))
        o = _COut(*[r[n].ctypes.data if n in r else None for n, _ in _COut._fields_])
        self.ctx._check(self.ctx.L.cg_certify_empty_slot(self.h, u64(view), u64(seq), C.byref(o)))
        return r

    def fetch_ticket(self, ticket: int, want_outputs=False, want_leaves=False):
        """Results of an already certified ticket (its slot not yet reused),
        e.g. batch i read back while batch i+1's forwards run."""
        return self.fetch(want_outputs, want_leaves, _fetch_ticket=ticket)

    def fetch(self, want_outputs=False, want_leaves=False, _enqueue=None,
              _outputs=None, _ticket=None, _fetch_ticket=None):
        B = self._lastB if _fetch_ticket is None else self._doneB[_fetch_ticket]
        N, v, k = self.N, self.v, self.topk
        amax = N * B + B + N
        r = dict(selected=np.zeros(B, np.uint32), diameter=np.zeros(B),
                 satisfied=np.zeros(B, np.uint8), label=np.zeros(B, np.int64),
                 r_roots=np.zeros((N, 32), np.uint8), a_root=np.zeros(32, np.uint8),
                 manifest_len=np.zeros(1, np.uint64),
                 manifest_kind=np.zeros(amax, np.uint8),
                 manifest_node=np.zeros(amax, np.uint32),
                 manifest_op=np.zeros(amax, np.uint32),
                 a_leaf_hashes=np.zeros((amax, 32), np.uint8))
        if want_leaves:
            r["leaf_hashes"] = np.zeros((N, B, 32), np.uint8)
        if want_outputs:
            r["outputs"] = np.zeros((N, B, v), np.float64)
            r["topk_idx"] = np.zeros((N, B, k), np.uint32)
            r["topk_val"] = np.zeros((N, B, k), np.float64)
        o = _COut(*[r[n].ctypes.data if n in r else None
                    for n, _ in _COut._fields_])
        if _ticket is not None:
            rc = self.ctx.L.cg_certify_ticket(self.h, C.c_uint64(_ticket), C.byref(o))
        elif _outputs is not None:
            rc = self.ctx.L.cg_certify_outputs(self.h, C.byref(_enqueue[0]),
                                               _p(_outputs), C.byref(o))
        elif _enqueue is not None:
            rc = self.ctx.L.cg_certify_batch(self.h, C.byref(_enqueue[0]), C.byref(o))
        elif _fetch_ticket is not None:
            rc = self.ctx.L.cg_group_fetch_ticket(self.h, C.c_uint64(_fetch_ticket), C.byref(o))
        else:
            rc = self.ctx.L.cg_group_fetch(self.h, C.byref(o))
        self.ctx._check(rc)
        m = int(r["manifest_len"][0])
        for key in ("manifest_kind", "manifest_node", "manifest_op", "a_leaf_hashes"):
            r[key] = r[key][:m]
        r["satisfied"] = r["satisfied"].astype(bool)
        return r
