"""TEST INFRASTRUCTURE — ctypes front-end to the CPU checkers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module. It is
the checker, never the thing measured or shipped.

* :class:`Oracle` wraps ``oracle/liboracle.so`` — the plain-C restatement of
  the reference's hot-path algorithms (``oracle/credo_oracle.c``).
* :class:`Reference` wraps ``oracle/_ref/libcredo_ref.so`` — the unmodified
  reference library compiled in place (``oracle/Makefile``) plus the
  ``ref_capi.cpp`` shims. It exists only where it was built.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcredo_ref.so")
REF_SODIUM_SO = os.path.join(HERE, "_ref", "libcredo_ref_sodium.so")

u64 = C.c_uint64
u32 = C.c_uint32
dbl = C.c_double
vp = C.c_void_p


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def build_oracle() -> None:
    """Compile liboracle.so (plain C, gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            if not os.path.exists(ORACLE_SO):
                build_oracle()
            L = C.CDLL(ORACLE_SO)
            L.oc_request_encode.restype = u64
            L.oc_result_encode.restype = u64
            L.oc_failure_leaf.restype = u64
            L.oc_ensemble_label.restype = C.c_int64
            L.oc_argmax.restype = u64
            L.oc_delta.restype = dbl
            L.oc_attest_manifest.restype = u64
            Oracle._lib = L
        self.L = Oracle._lib

    # -- SHA / merkle -----------------------------------------------------
    def sha256(self, data: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self.L.oc_sha256(data, u64(len(data)), out)
        return out.raw

    def midstate(self, data: bytes, nblocks: int) -> np.ndarray:
        out = np.zeros(8, np.uint32)
        self.L.oc_sha256_midstate(data, u64(nblocks), _p(out))
        return out

    def leaf_hash(self, leaf: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self.L.oc_leaf_hash(leaf, u64(len(leaf)), out)
        return out.raw

    def tagged_leaf_hash(self, tag: int, a: bytes, b: bytes = b"") -> bytes:
        out = C.create_string_buffer(32)
        self.L.oc_tagged_leaf_hash(C.c_uint8(tag), a, u64(len(a)), b,
                                   u64(len(b)), out)
        return out.raw

    def merkle_root(self, leaf_hashes: list[bytes]) -> bytes:
        buf = b"".join(leaf_hashes)
        out = C.create_string_buffer(32)
        rc = self.L.oc_merkle_root(buf, u64(len(leaf_hashes)), out)
        if rc != 0:
            raise ValueError("merkle: empty leaf list")
        return out.raw

    # -- encodings ----------------------------------------------------------
    def request_encode(self, req_id, gid: bytes, inp: np.ndarray, eps, pub,
                       nonce: bytes, sig) -> bytes:
        inp = np.ascontiguousarray(inp, np.float64)
        args = (req_id, gid, u64(len(gid)), _p(inp), u64(inp.size),
                C.c_int(eps is not None), dbl(eps or 0.0), pub, nonce,
                u64(len(nonce)), sig)
        n = self.L.oc_request_encode(*args, None)
        out = C.create_string_buffer(n)
        self.L.oc_request_encode(*args, out)
        return out.raw

    def hash_ops(self, encs: list[bytes], versions, statuses, reasons=None) -> bytes:
        """hash_ops (messages.cpp:197-202): H(0x4F || u32be n || per op
        OpEntry::encode (messages.cpp:161-169) = u8 kind 0 || bool 1 ||
        request encoding || bool 0 || u64be version || u8 status || str
        reason)."""
        parts = [b"\x4f", struct.pack(">I", len(encs))]
        for i, e in enumerate(encs):
            r = (reasons[i] if reasons is not None else "").encode()
            parts += [b"\x00\x01", e, b"\x00", struct.pack(">QB", int(versions[i]), int(statuses[i])),
                      struct.pack(">I", len(r)), r]
        return self.sha256(b"".join(parts))

    def result_encode(self, req_id, node, gid: bytes, version, out_vec,
                      model_digest) -> bytes:
        o = np.ascontiguousarray(out_vec, np.float64)
        args = (req_id, u64(node), gid, u64(len(gid)), u64(version), _p(o),
                u64(o.size), model_digest)
        n = self.L.oc_result_encode(*args, None)
        out = C.create_string_buffer(n)
        self.L.oc_result_encode(*args, out)
        return out.raw

    def failure_leaf(self, req_id, gid: bytes, version,
                     reason=b"quorum unsatisfied") -> bytes:
        args = (req_id, gid, u64(len(gid)), u64(version), reason,
                u64(len(reason)))
        n = self.L.oc_failure_leaf(*args, None)
        out = C.create_string_buffer(n)
        self.L.oc_failure_leaf(*args, out)
        return out.raw

    # -- agreement ----------------------------------------------------------
    def select_quorum(self, outs: np.ndarray, node_idx, n, f, metric, eps):
        outs = np.ascontiguousarray(outs, np.float64)
        idx = np.ascontiguousarray(node_idx, np.uint64)
        mask, diam, sat = u64(), dbl(), C.c_int()
        rc = self.L.oc_select_quorum(_p(outs), _p(idx), u64(outs.shape[0]),
                                     u64(outs.shape[1]), u64(n), u64(f),
                                     u32(metric), dbl(eps), C.byref(mask),
                                     C.byref(diam), C.byref(sat))
        if rc != 0:
            raise ValueError("select_quorum: invalid argument")
        return mask.value, diam.value, bool(sat.value)

    def delta(self, metric, x, y) -> float:
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        return self.L.oc_delta(u32(metric), _p(x), _p(y), u64(x.size))

    def ensemble_label(self, outs: np.ndarray, mask: int, f: int) -> int:
        outs = np.ascontiguousarray(outs, np.float64)
        return self.L.oc_ensemble_label(_p(outs), u64(outs.shape[0]),
                                        u64(outs.shape[1]), u64(mask), u64(f))

    def label_digest(self, req_id: bytes, version: int, label: int) -> bytes:
        out = C.create_string_buffer(32)
        self.L.oc_label_digest(req_id, u64(version), C.c_int64(label), out)
        return out.raw

    def agree_batch(self, outs: np.ndarray, f: int, metric: int, eps, req_ids=None,
                    version: int = 0):
        """outs (n, R, v): per request select_quorum + ensemble_label (+ the
        compact label digests when req_ids (R, 32) are given)."""
        outs = np.ascontiguousarray(outs, np.float64)
        n, R, v = outs.shape
        eps = np.ascontiguousarray(np.broadcast_to(eps, (R,)), np.float64)
        sel = np.zeros(R, np.uint64)
        diam = np.zeros(R)
        sat = np.zeros(R, np.uint8)
        lab = np.zeros(R, np.int64)
        dig = np.zeros((R, 32), np.uint8)
        ids = None if req_ids is None else np.ascontiguousarray(req_ids, np.uint8)
        rc = self.L.oc_agree_batch(_p(outs), u64(R), u64(n), u64(f), u64(v), u32(metric),
                                   _p(eps), None if ids is None else _p(ids), u64(version),
                                   _p(sel), _p(diam), _p(sat), _p(lab),
                                   None if ids is None else _p(dig))
        if rc != 0:
            raise ValueError("select_quorum: invalid argument")
        return dict(selected=sel.astype(np.uint32), diameter=diam, satisfied=sat.astype(bool),
                    label=lab, digest=dig if ids is not None else None)

    def argmax(self, v) -> int:
        v = np.ascontiguousarray(v, np.float64)
        return self.L.oc_argmax(_p(v), u64(v.size))

    def topk(self, v, k):
        v = np.ascontiguousarray(v, np.float64)
        idx = np.zeros(k, np.uint32)
        val = np.zeros(k, np.float64)
        self.L.oc_topk(_p(v), u64(v.size), u32(k), _p(idx), _p(val))
        return idx, val

    def linear_run(self, W, b, x, softmax: bool) -> np.ndarray:
        W = np.ascontiguousarray(W, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        v, u = W.shape
        y = np.zeros(v, np.float64)
        self.L.oc_linear_run(_p(W), _p(b), u64(u), u64(v), C.c_int(softmax),
                             _p(x), _p(y))
        return y

    def perturb(self, node: int, model_digest: bytes, x, y, mag: float) -> np.ndarray:
        """PerturbingExecutor::run's offset for one request (model.cpp:82-105)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.array(y, np.float64)
        self.L.oc_perturb(u64(node), bytes(model_digest), _p(x), u64(x.size),
                          _p(y), u64(y.size), C.c_double(mag))
        return y

    def softmax(self, y) -> np.ndarray:
        y = np.array(y, np.float64)
        self.L.oc_softmax(_p(y), u64(y.size))
        return y

    def attest_manifest(self, sel_mask, satisfied, N):
        sel = np.ascontiguousarray(sel_mask, np.uint64)
        sat = np.ascontiguousarray(satisfied, np.uint8)
        B = sel.size
        cap = N * B + B + N
        kinds = np.zeros(cap, np.uint8)
        nodes = np.zeros(cap, np.uint64)
        ops = np.zeros(cap, np.uint64)
        n = self.L.oc_attest_manifest(u64(B), u64(N), _p(sel), _p(sat),
                                      _p(kinds), _p(nodes), _p(ops))
        return [(int(kinds[i]), int(nodes[i]), int(ops[i])) for i in range(n)]


def parse_linear_model_file(buf: bytes):
    """Decode LinearToyModel::to_file_bytes (model.cpp:38-46)."""
    import struct
    i, o = struct.unpack(">QQ", buf[:16])
    sm = buf[16]
    n = struct.unpack(">I", buf[17:21])[0]
    W = np.frombuffer(buf[21:21 + 8 * n], dtype=">f8").astype(np.float64)
    off = 21 + 8 * n
    nb = struct.unpack(">I", buf[off:off + 4])[0]
    b = np.frombuffer(buf[off + 4:off + 4 + 8 * nb], dtype=">f8").astype(np.float64)
    return int(i), int(o), bool(sm), W.reshape(o, i), b


def parse_request(buf: bytes):
    """Decode InferenceRequest::encode (domain.cpp:153-175) into fields."""
    import struct
    off = 0
    req_id = buf[0:32]; off = 32
    gl = struct.unpack(">I", buf[off:off + 4])[0]; off += 4
    gid = buf[off:off + gl]; off += gl
    n = struct.unpack(">I", buf[off:off + 4])[0]; off += 4
    inp = np.frombuffer(buf[off:off + 8 * n], dtype=">f8").astype(np.float64); off += 8 * n
    has = buf[off]; off += 1
    eps = None
    if has:
        eps = struct.unpack(">d", buf[off:off + 8])[0]; off += 8
    pub = buf[off:off + 32]; off += 32
    nl = struct.unpack(">I", buf[off:off + 4])[0]; off += 4
    nonce = buf[off:off + nl]; off += nl
    sig = buf[off:off + 64]; off += 64
    assert off == len(buf)
    return dict(request_id=req_id, group_id=gid, input=inp, eps=eps, pub=pub,
                nonce=nonce, sig=sig)


class Reference:
    """The compiled reference (oracle/_ref). Raises OSError when absent.
    backend "openssl": SHA-256 through the OpenSSL shim (SHA-NI);
    "libsodium": the reference's own shipped libsodium crypto_hash_sha256
    (identical digests, ~50x slower)."""
    _libs = {}

    @staticmethod
    def available(backend: str = "openssl") -> bool:
        return os.path.exists(REF_SO if backend == "openssl" else REF_SODIUM_SO)

    def __init__(self, backend: str = "openssl"):
        if backend not in Reference._libs:
            L = C.CDLL(REF_SO if backend == "openssl" else REF_SODIUM_SO)
            L.ref_model_file_len.restype = u64
            L.ref_request_len.restype = u64
            L.ref_ensemble_label.restype = C.c_int64
            L.ref_batch_new.restype = vp
            L.ref_batch_new.argtypes = [vp, vp, u64, u64]
            L.ref_batch_free.argtypes = [vp]
            Reference._libs[backend] = L
        self.L = Reference._libs[backend]

    def sha256(self, data: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self.L.ref_sha256(data, u64(len(data)), out)
        return out.raw

    def leaf_hash(self, leaf: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self.L.ref_leaf_hash(leaf, u64(len(leaf)), out)
        return out.raw

    def merkle_root(self, leaves: list[bytes]) -> bytes:
        lens = np.array([len(x) for x in leaves], np.uint64)
        out = C.create_string_buffer(32)
        rc = self.L.ref_merkle_root(b"".join(leaves), _p(lens),
                                    u64(len(leaves)), out)
        if rc != 0:
            raise ValueError("merkle: empty leaf list")
        return out.raw

    def generate_group(self, gid: bytes, u, v, models, metric, eps, seed,
                       salt=0, softmax=False):
        flen = self.L.ref_model_file_len(u64(u), u64(v))
        files = C.create_string_buffer(flen * models)
        digs = C.create_string_buffer(32 * models)
        rc = self.L.ref_generate_group(gid, u64(u), u64(v), u64(models),
                                       u32(metric), dbl(eps), u64(seed),
                                       u64(salt), C.c_int(int(softmax)),
                                       files, digs)
        assert rc == 0, rc
        return ([files.raw[i * flen:(i + 1) * flen] for i in range(models)],
                [digs.raw[32 * i:32 * i + 32] for i in range(models)])

    def make_requests(self, scenario_seed, workload_seed, n, u, gid: bytes):
        rl = self.L.ref_request_len(u64(len(gid)), u64(u), u64(16), 0)
        inputs = np.zeros((n, u), np.float64)
        enc = C.create_string_buffer(rl * n)
        rc = self.L.ref_make_requests(u64(scenario_seed), u64(workload_seed),
                                      u64(n), u64(u), gid, _p(inputs), enc)
        assert rc == 0, rc
        return inputs, [enc.raw[i * rl:(i + 1) * rl] for i in range(n)]

    def make_request(self, key_seed, nonce: bytes, gid: bytes, inp, eps=None):
        inp = np.ascontiguousarray(inp, np.float64)
        cap = 200 + 8 * inp.size + len(nonce) + len(gid)
        out = C.create_string_buffer(cap)
        ln = u64()
        rc = self.L.ref_make_request(u64(key_seed), nonce, u64(len(nonce)), gid,
                                     _p(inp), u64(inp.size),
                                     C.c_int(eps is not None), dbl(eps or 0.0),
                                     out, u64(cap), C.byref(ln))
        assert rc == 0, rc
        return out.raw[:ln.value]

    def verify_request(self, enc: bytes) -> int:
        return self.L.ref_verify_request(enc, u64(len(enc)))

    def auth_path(self, leaves: list[bytes], index: int):
        """Tree::build(leaves).auth_path(index) -> [(sibling, side)]."""
        lens = np.array([len(x) for x in leaves], np.uint64)
        sib = C.create_string_buffer(32 * 64)
        sides = C.create_string_buffer(64)
        k = self.L.ref_auth_path(b"".join(leaves), _p(lens), u64(len(leaves)), u64(index),
                                 sib, sides)
        assert k >= 0
        return [(sib.raw[32 * i:32 * i + 32], sides.raw[i]) for i in range(k)]

    def path_root(self, leaf: bytes, path) -> bytes:
        """merkle::get_merkle_root(path, leaf)."""
        sib = b"".join(s for s, _ in path) or b"\0"
        sides = bytes(d for _, d in path) or b"\0"
        out = C.create_string_buffer(32)
        assert self.L.ref_path_root(leaf, u64(len(leaf)), sib, sides, C.c_uint32(len(path)),
                                    out) == 0
        return out.raw

    def hash_ops(self, encs: list[bytes], versions, statuses, reasons=None) -> bytes:
        """messages.cpp:197-202 over request ops."""
        lens = np.array([len(e) for e in encs], np.uint64)
        ver = np.ascontiguousarray(versions, np.uint64)
        st = np.ascontiguousarray(statuses, np.uint8)
        rs = None
        if reasons is not None:
            rs = (C.c_char_p * len(reasons))(*[r.encode() for r in reasons])
        out = C.create_string_buffer(32)
        assert self.L.ref_hash_ops(b"".join(encs), _p(lens), u64(len(encs)), _p(ver), _p(st),
                                   rs, out) == 0
        return out.raw

    def certify_slot(self, encs, kinds, reasons, N, f, eps, outputs, version, digests):
        """A mixed PRE-PREPARE op list (ok / rejected requests, activate_group
        ops) through build_result_tree + the try_attest manifest; returns the
        roots, manifest length, satisfied flags, every op's OpEntry encoding
        and the rejected ops' FailureRecord encodings."""
        B = len(kinds)
        lens = np.array([len(e) for e in encs], np.uint64)
        k8 = np.ascontiguousarray(kinds, np.uint8)
        rs = (C.c_char_p * B)(*[r.encode() for r in reasons])
        o = np.ascontiguousarray(outputs, np.float64)
        cap = 1 << 21
        ent = np.zeros(B * cap, np.uint8)
        rec = np.zeros(B * cap, np.uint8)
        el = np.zeros(B, np.uint64)
        rl = np.zeros(B, np.uint64)
        rr = C.create_string_buffer(32 * N)
        ar = C.create_string_buffer(32)
        ml = u64()
        sat = np.zeros(B, np.uint8)
        rc = self.L.ref_certify_slot(b"".join(encs) or b"\0", _p(lens), u64(B), _p(k8), rs, u64(N),
                                     u64(f), dbl(eps), _p(o), u64(o.shape[2]), u64(version),
                                     b"".join(digests), rr, ar, C.byref(ml), _p(sat), _p(ent),
                                     _p(el), _p(rec), _p(rl), u64(cap))
        assert rc == 0, rc
        return dict(r_roots=[rr.raw[32 * i:32 * i + 32] for i in range(N)], a_root=ar.raw,
                    manifest_len=ml.value, satisfied=sat,
                    entries=[ent[k * cap:k * cap + int(el[k])].tobytes() for k in range(B)],
                    records=[rec[k * cap:k * cap + int(rl[k])].tobytes() for k in range(B)])

    def signing_digest(self, enc: bytes) -> bytes:
        out = C.create_string_buffer(32)
        assert self.L.ref_signing_digest(enc, u64(len(enc)), out) == 0
        return out.raw

    def linear_run(self, file: bytes, inputs: np.ndarray, v: int) -> np.ndarray:
        x = np.ascontiguousarray(inputs, np.float64)
        y = np.zeros((x.shape[0], v), np.float64)
        rc = self.L.ref_linear_run(file, u64(len(file)), _p(x),
                                   u64(x.shape[0]), _p(y))
        assert rc == 0, rc
        return y

    def perturbing_run(self, file: bytes, inputs: np.ndarray, v: int, node: int,
                       magnitude: float) -> np.ndarray:
        x = np.ascontiguousarray(inputs, np.float64)
        y = np.zeros((x.shape[0], v), np.float64)
        rc = self.L.ref_perturbing_run(file, u64(len(file)), _p(x), u64(x.shape[0]),
                                       u64(node), C.c_double(magnitude), _p(y))
        if rc == -2:
            raise ValueError("negative magnitude")
        assert rc == 0, rc
        return y

    def select_quorum(self, outs, node_idx, n, f, metric, eps):
        outs = np.ascontiguousarray(outs, np.float64)
        idx = np.ascontiguousarray(node_idx, np.uint64)
        mask, diam, sat = u64(), dbl(), C.c_int()
        rc = self.L.ref_select_quorum(_p(outs), _p(idx), u64(outs.shape[0]),
                                      u64(outs.shape[1]), u64(n), u64(f),
                                      u32(metric), dbl(eps), C.byref(mask),
                                      C.byref(diam), C.byref(sat))
        if rc != 0:
            raise ValueError("select_quorum: invalid argument")
        return mask.value, diam.value, bool(sat.value)

    def ensemble_label(self, outs, mask, f) -> int:
        outs = np.ascontiguousarray(outs, np.float64)
        return self.L.ref_ensemble_label(_p(outs), u64(outs.shape[0]),
                                         u64(outs.shape[1]), u64(mask), u64(f))

    def result_leaf_hash(self, req_enc: bytes, node, gid: bytes, version,
                         out_vec, model_digest: bytes) -> bytes:
        o = np.ascontiguousarray(out_vec, np.float64)
        out = C.create_string_buffer(32)
        rc = self.L.ref_result_leaf_hash(req_enc, u64(len(req_enc)), u64(node),
                                         gid, u64(version), _p(o), u64(o.size),
                                         model_digest, out)
        assert rc == 0, rc
        return out.raw

    # -- batch certification (CPU baseline) ---------------------------------
    def batch_new(self, encs: list[bytes], version: int):
        lens = np.array([len(e) for e in encs], np.uint64)
        buf = b"".join(encs)
        self._keep = buf
        h = self.L.ref_batch_new(C.c_char_p(buf), _p(lens), len(encs), version)
        assert h
        return h

    def batch_free(self, h):
        self.L.ref_batch_free(h)

    def certify_batch(self, h, N, f, metric, eps, outputs, version,
                      model_digests: list[bytes], threads=1, view=0, seq=1, missing=None):
        """outputs: (N, B, v) float64; missing: optional B flags (request has
        no result from any provider: a misfit)."""
        outputs = np.ascontiguousarray(outputs, np.float64)
        N_, B, v = outputs.shape
        sel = np.zeros(B, np.uint64)
        diam = np.zeros(B, np.float64)
        sat = np.zeros(B, np.uint8)
        label = np.zeros(B, np.int64)
        r_roots = C.create_string_buffer(32 * N)
        a_root = C.create_string_buffer(32)
        mlen = u64()
        miss = None if missing is None else np.ascontiguousarray(missing, np.uint8)
        rc = self.L.ref_certify_batch_ex(
            vp(h), u64(N), u64(f), u32(metric), dbl(eps), _p(outputs), u64(v),
            u64(version), b"".join(model_digests), u64(view), u64(seq),
            C.c_int(threads), _p(sel), _p(diam), _p(sat), _p(label), r_roots,
            a_root, C.byref(mlen), _p(miss))
        assert rc == 0, rc
        return dict(sel_mask=sel, diameter=diam, satisfied=sat, label=label,
                    r_roots=[r_roots.raw[32 * i:32 * i + 32] for i in range(N)],
                    a_root=a_root.raw, manifest_len=mlen.value)
