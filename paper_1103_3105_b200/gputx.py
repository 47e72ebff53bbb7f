"""ctypes binding of include/gputx.h — argument marshalling only.

The names mirror the C ABI (gputx_open_db / load_column / seal / register_types /
submit_bulk / execute / read_results ...).  No transaction logic lives here.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "libgputx.so")

GPUTX_TPL, GPUTX_PART, GPUTX_KSET, GPUTX_AUTO, GPUTX_TPL_RELAXED, GPUTX_PART_RELAXED = 0, 1, 2, 3, 4, 5
TPL, PART, KSET, AUTO, TPL_RELAXED, PART_RELAXED = "tpl", "part", "kset", "auto", "tpl_relaxed", "part_relaxed"
STRATEGIES = {TPL: GPUTX_TPL, PART: GPUTX_PART, KSET: GPUTX_KSET, AUTO: GPUTX_AUTO, TPL_RELAXED: GPUTX_TPL_RELAXED,
              PART_RELAXED: GPUTX_PART_RELAXED}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "EDUP_TYPE", 4: "EUNKNOWN_TYPE", 5: "ESTATE",
                6: "ECAPACITY", 7: "ECROSS", 8: "EDEADLOCK", 9: "ECUDA", 10: "ENCCL"}
OUT_STRIDE = {1: 8, 2: 40, 3: 200, 4: 4}
FLAG_ADD_RULE = 1            # include/gputx.h GPUTX_FLAG_ADD_RULE
FLAG_PACKED_OUT = 2          # include/gputx.h GPUTX_FLAG_PACKED_OUT
FLAG_DEFERRED_CHECK = 4      # include/gputx.h GPUTX_FLAG_DEFERRED_CHECK


class GputxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class Config(ctypes.Structure):
    _fields_ = [("schema", ctypes.c_int), ("dims", ctypes.c_uint32 * 4), ("max_bulk", ctypes.c_uint64),
                ("insert_capacity", ctypes.c_uint64), ("part_size", ctypes.c_uint32), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint32), ("shard", ctypes.c_uint32),
                ("nshards", ctypes.c_uint32), ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p)]


def torch_allocator(device: int):
    """(alloc, free) callbacks routing the engine's device memory through PyTorch's caching
    allocator (include/gputx.h gputx_alloc_fn) -- memory plumbing only."""
    import torch

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream or None)
        except Exception:
            return None

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(ptr)

    return ALLOC_FN(_alloc), FREE_FN(_free)


class BulkC(ctypes.Structure):
    _fields_ = [("type", ctypes.c_void_p), ("param_off", ctypes.c_void_p), ("param_words", ctypes.c_void_p),
                ("n", ctypes.c_uint64), ("on_device", ctypes.c_int), ("ts", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("n", "committed", "aborted", "depth", "ksets", "zero_set", "records",
                                               "rank_passes", "parts", "fragments", "max_chain", "launches")] + \
               [(k, ctypes.c_double) for k in ("ms_emit", "ms_sort", "ms_rank", "ms_group", "ms_exec", "ms_merge",
                                               "ms_total")] + \
               [(k, ctypes.c_uint64) for k in ("cross", "strategy")] + \
               [(k, ctypes.c_double) for k in ("ms_ingest", "ms_exchange")] + [("flags", ctypes.c_uint64),
                                                                                   ("out_bytes", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["strategy"] = STRATEGY_NAMES[d["strategy"]]
        return d


_lib = None


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libgputx.so (build it first with paper_1103_3105_b200.build.build()).
    Raises if it is missing: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built; run python -m paper_1103_3105_b200.build")
    lib = ctypes.CDLL(_LIB_PATH)
    P, U32, U64, I = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sig = {
        "gputx_open_db": ([ctypes.POINTER(Config), ctypes.POINTER(P)], I),
        "gputx_load_column": ([P, ctypes.c_char_p, P, U64], I),
        "gputx_column_info": ([P, U32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(U32), ctypes.POINTER(U64)], I),
        "gputx_seal": ([P], I),
        "gputx_register_types": ([P, P, U32], I),
        "gputx_set_grouping": ([P, U32], I),
        "gputx_pool_submit": ([P, P, P], I),
        "gputx_pool_step": ([P, P, P], I),
        "gputx_pool_read": ([P, P, P, P, U64, P], I),
        "gputx_pool_pending": ([P, P], I),
        "gputx_read_serial_order": ([P, P, U64], I),
        "gputx_snapshot": ([P, P, P], I),
        "gputx_run_bulks": ([P, P, U64, I, P, P, P], I),
        "gputx_shard_export": ([P, P], I),
        "gputx_shard_connect": ([P, P], I),
        "gputx_shard_connect_local": ([P, U32], I),
        "gputx_shard_dispatch": ([P, P], I),
        "gputx_shard_receive": ([P, P], I),
        "gputx_shard_return": ([P], I),
        "gputx_shard_collect": ([P], I),
        "gputx_submit_bulk": ([P, ctypes.POINTER(BulkC), ctypes.POINTER(U64)], I),
        "gputx_execute": ([P, I, ctypes.POINTER(Stats)], I),
        "gputx_execute_async": ([P, I], I),
        "gputx_wait": ([P, ctypes.POINTER(Stats)], I),
        "gputx_read_results": ([P, P, P, U64], I),
        "gputx_read_out_offsets": ([P, P, U64, P], I),
        "gputx_results_device": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(U64)], I),
        "gputx_out_stride": ([I], U32),
        "gputx_read_column": ([P, ctypes.c_char_p, P, U64], I),
        "gputx_insert_rows": ([P, ctypes.c_char_p, ctypes.POINTER(U64)], I),
        "gputx_read_insert_column": ([P, ctypes.c_char_p, ctypes.c_char_p, P, U64], I),
        "gputx_read_depths": ([P, P, U64], I),
        "gputx_read_perm": ([P, P, U64], I),
        "gputx_reset": ([P], I),
        "gputx_close_db": ([P], None),
        "gputx_last_error": ([P], ctypes.c_char_p),
        "gputx_set_launch": ([P, U32, U32, U32], I),
        "gputx_set_chooser": ([P, U64, U64, U64], I),
        "gputx_trace_rounds": ([P, I], I),
        "gputx_read_round_ns": ([P, P, U64], I),
        "gputx_read_rank_ns": ([P, P, U64], I),
        "gputx_shard_stride": ([I, I], U32),
        "gputx_shard_pack": ([P, ctypes.POINTER(BulkC), P, U64, P], I),
        "gputx_shard_submit": ([P, P, U64, ctypes.POINTER(U64)], I),
        "gputx_shard_return_pack": ([P, P, U64, P], I),
        "gputx_shard_return_merge": ([P, P, U64], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


EXPORTED = ["gputx_open_db", "gputx_load_column", "gputx_column_info", "gputx_seal", "gputx_register_types",
            "gputx_submit_bulk", "gputx_execute", "gputx_execute_async", "gputx_wait", "gputx_read_results", "gputx_results_device",
            "gputx_out_stride", "gputx_read_column", "gputx_insert_rows", "gputx_read_insert_column",
            "gputx_read_depths", "gputx_read_perm", "gputx_reset", "gputx_close_db", "gputx_last_error",
            "gputx_set_launch", "gputx_set_chooser", "gputx_trace_rounds", "gputx_read_round_ns",
            "gputx_read_rank_ns", "gputx_shard_stride", "gputx_shard_pack", "gputx_shard_submit",
            "gputx_shard_return_pack", "gputx_shard_return_merge", "gputx_set_grouping",
            "gputx_pool_submit", "gputx_pool_step", "gputx_pool_read", "gputx_pool_pending",
            "gputx_read_serial_order", "gputx_snapshot", "gputx_run_bulks", "gputx_shard_export",
            "gputx_shard_connect", "gputx_shard_connect_local", "gputx_shard_dispatch", "gputx_shard_receive",
            "gputx_shard_return", "gputx_shard_collect", "gputx_read_out_offsets"]
PEER_BLOB_BYTES = 128                    # include/gputx.h GPUTX_PEER_BLOB_BYTES

INSERT_TABLES = {
    1: {"history": ["h_tid", "h_bid", "h_aid", "h_delta", "h_ts"]},
    2: {},
    4: {},
    3: {"order": ["o_id", "o_d", "o_w", "o_c", "o_entry_d", "o_ol_cnt", "o_all_local"],
        "new_order": ["no_o_id", "no_d", "no_w"],
        "order_line": ["ol_o_id", "ol_d", "ol_w", "ol_number", "ol_i_id", "ol_supply_w", "ol_quantity", "ol_amount"],
        "history": ["h_c", "h_cd", "h_cw", "h_d", "h_w", "h_date", "h_amount"]},
}
SIGNED_INSERT_COLS = {"h_delta", "ol_amount", "h_amount"}


def unpack_outputs(buf: np.ndarray, off: np.ndarray, stride: int) -> np.ndarray:
    """Packed output records (GPUTX_FLAG_PACKED_OUT) -> u8[n, stride] (zero-padded)."""
    n = len(off) - 1
    out = np.zeros((n, stride), np.uint8)
    size = np.diff(off.astype(np.int64))
    for s in np.unique(size):
        if s == 0:
            continue
        rows = np.nonzero(size == s)[0]
        out[rows, :s] = buf[off[rows].astype(np.int64)[:, None] + np.arange(s)]
    return out


def _ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    assert a.flags.c_contiguous
    return a.ctypes.data


class Database:
    """One gputx_db handle: an HBM-resident database of one schema on one GPU."""

    def __init__(self, schema: int, dims, max_bulk: int, image: dict | None = None, *, part_size: int = 0,
                 device: int = 0, stream: int | None = None, insert_capacity: int = 0, shard: int = 0,
                 nshards: int = 1, add_rule: bool = False, torch_memory: bool = False, packed_out: bool = False,
                 deferred_check: bool = False):
        self.lib = load_library()
        self.schema = schema
        cfg = Config()
        cfg.schema = schema
        for k, v in enumerate(dims):
            cfg.dims[k] = int(v)
        cfg.max_bulk = int(max_bulk)
        cfg.insert_capacity = int(insert_capacity)
        cfg.part_size = int(part_size)
        cfg.device = int(device)
        cfg.stream = stream
        cfg.flags = ((FLAG_ADD_RULE if add_rule else 0) | (FLAG_PACKED_OUT if packed_out else 0) |
                     (FLAG_DEFERRED_CHECK if deferred_check else 0))
        self.packed = bool(packed_out)
        cfg.shard = int(shard)
        cfg.nshards = int(nshards)
        if torch_memory:                     # device memory from PyTorch's caching allocator
            self._alloc_cbs = torch_allocator(int(device))
            cfg.alloc, cfg.free = self._alloc_cbs
        self.shard, self.nshards, self.device = int(shard), int(nshards), int(device)
        self._bufs = {}
        h = ctypes.c_void_p()
        self._check(self.lib.gputx_open_db(ctypes.byref(cfg), ctypes.byref(h)), None)
        self.h = h
        self.stride = OUT_STRIDE[schema]
        self.n = 0
        self.columns = {}
        k = 0
        while True:
            nm, el, cnt = ctypes.c_char_p(), ctypes.c_uint32(), ctypes.c_uint64()
            if self.lib.gputx_column_info(self.h, k, ctypes.byref(nm), ctypes.byref(el), ctypes.byref(cnt)) != 0:
                break
            self.columns[nm.value.decode()] = (el.value, cnt.value)
            k += 1
        if image is not None:
            for name in self.columns:
                self.load_column(name, image[name])
            self.seal()

    # --------------------------------------------------------------------------------
    def _check(self, status: int, h):
        if status != 0:
            msg = self.lib.gputx_last_error(h).decode() if h else "open failed"
            raise GputxError(status, msg)

    def load_column(self, name: str, arr: np.ndarray):
        a = np.ascontiguousarray(arr)
        self._check(self.lib.gputx_load_column(self.h, name.encode(), a.ctypes.data, a.nbytes), self.h)

    def seal(self):
        self._check(self.lib.gputx_seal(self.h), self.h)

    def register_types(self, ids):
        a = np.ascontiguousarray(np.asarray(ids, np.uint32))
        self._check(self.lib.gputx_register_types(self.h, a.ctypes.data if a.size else None, a.size), self.h)

    def _bulk(self, bulk, type, param_off, param_words, ts, on_device) -> BulkC:
        if bulk is not None:
            type, param_off, param_words = bulk.type, bulk.param_off, bulk.param_words
            if ts is None:
                ts = getattr(bulk, "ts", None)
        if not on_device:
            type = np.ascontiguousarray(type, np.uint8)
            param_off = np.ascontiguousarray(param_off, np.uint32)
            param_words = np.ascontiguousarray(param_words, np.uint32)
            if param_words.size == 0:
                param_words = np.zeros(1, np.uint32)
            if ts is not None:
                ts = np.ascontiguousarray(ts, np.uint32)
        self._keep = (type, param_off, param_words, ts)
        return BulkC(_ptr(type), _ptr(param_off), _ptr(param_words), int(type.shape[0]), int(on_device),
                     _ptr(ts) if ts is not None and int(type.shape[0]) else None)

    def submit(self, bulk=None, *, type=None, param_off=None, param_words=None, ts=None,
               on_device: bool = False) -> int:
        """Submit a bulk: any object with .type/.param_off/.param_words (numpy, host), or
        the three arrays as torch CUDA tensors with on_device=True (resident in HBM).
        ts: optional global timestamps (u32, increasing)."""
        b = self._bulk(bulk, type, param_off, param_words, ts, on_device)
        first = ctypes.c_uint64()
        self._check(self.lib.gputx_submit_bulk(self.h, ctypes.byref(b), ctypes.byref(first)), self.h)
        self.n = int(b.n)
        return first.value

    # ---- sharding (include/gputx.h "Sharding") --------------------------------------
    def shard_stride(self, result: bool = False) -> int:
        return int(self.lib.gputx_shard_stride(self.schema, int(result)))

    def _buf(self, key: str, words: int):
        """A device u32 buffer (torch, on this handle's GPU) of at least `words` words."""
        import torch
        b = self._bufs.get(key)
        if b is None or b.numel() < words:
            b = torch.empty(max(words, 1024), dtype=torch.int32, device=f"cuda:{self.device}")
            self._bufs[key] = b
        return b

    def _packed(self, fn, key: str, stride: int, est: int):
        counts = (ctypes.c_uint64 * self.nshards)()
        send = self._buf(key, est * stride)
        st = fn(send, send.numel() // stride, counts)
        if st == 6:                      # ECAPACITY: counts are filled; grow and repack
            send = self._buf(key, sum(counts) * stride)
            st = fn(send, send.numel() // stride, counts)
        self._check(st, self.h)
        return send, [int(c) for c in counts]

    def shard_pack(self, bulk=None, *, type=None, param_off=None, param_words=None, ts=None,
                   on_device: bool = False):
        """Stage the home bulk; returns (send buffer, records per destination shard)."""
        b = self._bulk(bulk, type, param_off, param_words, ts, on_device)
        self.nh = int(b.n)
        stride = self.shard_stride(False)
        return self._packed(lambda buf, cap, c: self.lib.gputx_shard_pack(self.h, ctypes.byref(b), _ptr(buf), cap,
                                                                          ctypes.addressof(c)),
                            "send", stride, max(1024, self.nh // 4))

    def shard_submit(self, recv, n_recv: int) -> int:
        nl = ctypes.c_uint64()
        self._check(self.lib.gputx_shard_submit(self.h, _ptr(recv) if n_recv else None, int(n_recv),
                                                ctypes.byref(nl)), self.h)
        self.n_local = int(nl.value)
        self.n = self.nh
        return self.n_local

    def shard_return_pack(self):
        stride = self.shard_stride(True)
        return self._packed(lambda buf, cap, c: self.lib.gputx_shard_return_pack(self.h, _ptr(buf), cap,
                                                                                 ctypes.addressof(c)),
                            "ret", stride, max(1024, self.n_local // 4))

    def shard_return_merge(self, recv, n_recv: int):
        self._check(self.lib.gputx_shard_return_merge(self.h, _ptr(recv) if n_recv else None, int(n_recv)), self.h)

    # ---- fused peer-memory exchange (include/gputx.h "FUSED into the library") -----------
    def shard_export(self) -> bytes:
        buf = ctypes.create_string_buffer(PEER_BLOB_BYTES)
        self._check(self.lib.gputx_shard_export(self.h, buf), self.h)
        return buf.raw

    def shard_connect(self, blobs: list[bytes]):
        raw = b"".join(blobs)
        self._check(self.lib.gputx_shard_connect(self.h, raw), self.h)

    @staticmethod
    def shard_connect_local(dbs: list["Database"]):
        lib = dbs[0].lib
        arr = (ctypes.c_void_p * len(dbs))(*[d.h.value for d in dbs])
        st = lib.gputx_shard_connect_local(arr, len(dbs))
        if st != 0:
            raise GputxError(st, lib.gputx_last_error(dbs[0].h).decode())

    def shard_dispatch(self, bulk=None, *, type=None, param_off=None, param_words=None, ts=None,
                       on_device: bool = False):
        b = self._bulk(bulk, type, param_off, param_words, ts, on_device)
        self.nh = int(b.n)
        self._check(self.lib.gputx_shard_dispatch(self.h, ctypes.byref(b)), self.h)

    def shard_receive(self) -> int:
        nl = ctypes.c_uint64()
        self._check(self.lib.gputx_shard_receive(self.h, ctypes.byref(nl)), self.h)
        self.n_local = int(nl.value)
        self.n = self.nh
        return self.n_local

    def shard_return(self):
        self._check(self.lib.gputx_shard_return(self.h), self.h)

    def shard_collect(self):
        self._check(self.lib.gputx_shard_collect(self.h), self.h)

    def execute(self, strategy: str = KSET) -> dict:
        st = Stats()
        self._check(self.lib.gputx_execute(self.h, STRATEGIES[strategy], ctypes.byref(st)), self.h)
        return st.as_dict()

    def execute_async(self, strategy: str = KSET) -> None:
        """Enqueue the bulk's execution and return (complete it with wait())."""
        self._check(self.lib.gputx_execute_async(self.h, STRATEGIES[strategy]), self.h)

    def wait(self) -> dict:
        """Complete an execute_async: synchronise, raise its device-side errors, stats."""
        st = Stats()
        self._check(self.lib.gputx_wait(self.h, ctypes.byref(st)), self.h)
        return st.as_dict()

    # ---- streaming K-SET pool (include/gputx.h "Streaming K-SET") -------------------
    def pool_submit(self, bulk=None, *, type=None, param_off=None, param_words=None, on_device: bool = False) -> int:
        """Append arrivals to the transaction pool; returns the first assigned ts."""
        b = self._bulk(bulk, type, param_off, param_words, None, on_device)
        b.ts = None
        first = ctypes.c_uint64()
        self._check(self.lib.gputx_pool_submit(self.h, ctypes.byref(b), ctypes.byref(first)), self.h)
        return first.value

    def pool_step(self) -> dict:
        """Execute the pool's current 0-set; stats dict with n = executed transactions."""
        st = Stats()
        ex = ctypes.c_uint64()
        self._check(self.lib.gputx_pool_step(self.h, ctypes.byref(st), ctypes.byref(ex)), self.h)
        d = st.as_dict()
        d["executed"] = ex.value
        self.pool_last = ex.value
        return d

    def pool_read(self, cap: int | None = None):
        """(ts u32[n], status u8[n], out u8[n, stride]) of the last step's transactions."""
        n = ctypes.c_uint64()
        k = getattr(self, "pool_last", 0) if cap is None else cap
        ts = np.zeros(max(k, 1), np.uint32)
        st = np.zeros(max(k, 1), np.uint8)
        out = np.zeros((max(k, 1), self.stride), np.uint8)
        self._check(self.lib.gputx_pool_read(self.h, _ptr(ts), _ptr(st), _ptr(out), k, ctypes.byref(n)), self.h)
        m = n.value
        return ts[:m], st[:m], out[:m]

    def run_bulks(self, bulks, strategy: str = KSET, status=None, out=None, stats: bool = False):
        """gputx_run_bulks: host bulks back to back with overlapped H2D / D2H.  status / out:
        lists of caller-owned host arrays (u8[n_i], u8[n_i, stride]) or None."""
        k = len(bulks)
        arr = (BulkC * max(k, 1))()
        keep = []
        for i, b in enumerate(bulks):
            t = np.ascontiguousarray(b.type, np.uint8)
            po = np.ascontiguousarray(b.param_off, np.uint32)
            pw = np.ascontiguousarray(b.param_words, np.uint32)
            if pw.size == 0:
                pw = np.zeros(1, np.uint32)
            keep.append((t, po, pw))
            arr[i] = BulkC(_ptr(t), _ptr(po), _ptr(pw), int(t.shape[0]), 0, None)
        sp = (ctypes.c_void_p * max(k, 1))(*[(_ptr(a) if a is not None else None) for a in (status or [None] * k)])
        op = (ctypes.c_void_p * max(k, 1))(*[(_ptr(a) if a is not None else None) for a in (out or [None] * k)])
        sts = (Stats * max(k, 1))() if stats else None
        self._check(self.lib.gputx_run_bulks(self.h, arr, k, STRATEGIES[strategy], sp, op, sts), self.h)
        if k:
            self.n = int(bulks[-1].type.shape[0])
        self._keep = keep
        return [s.as_dict() for s in sts[:k]] if stats else None

    def snapshot(self) -> dict:
        """The current database via gputx_snapshot: {"columns": {name: bytes-view array},
        "tables": {table: {column: u32 array}}} (parsed from the documented layout)."""
        need = ctypes.c_uint64()
        self._check(self.lib.gputx_snapshot(self.h, None, ctypes.byref(need)), self.h)
        buf = np.zeros(need.value, np.uint8)
        self._check(self.lib.gputx_snapshot(self.h, _ptr(buf), ctypes.byref(need)), self.h)
        o = 0

        def take(k):
            nonlocal o
            v = buf[o:o + k]
            o += k
            return v

        def u32():
            return int(take(4).view(np.uint32)[0])

        def u64():
            return int(take(8).view(np.uint64)[0])

        assert bytes(take(8)) == b"GPTXSNAP" and u32() == 1
        res = {"schema": u32(), "dims": [u32() for _ in range(4)], "columns": {}, "tables": {}}
        ncols, ntab = u32(), u32()
        for _ in range(ncols):
            name = bytes(take(u32())).decode()
            el, cnt = u32(), u64()
            res["columns"][name] = take(el * cnt).copy()
        for _ in range(ntab):
            tname = bytes(take(u32())).decode()
            nc, rows = u32(), u64()
            res["tables"][tname] = {}
            for _ in range(nc):
                cname = bytes(take(u32())).decode()
                res["tables"][tname][cname] = take(rows * 4).copy().view(np.uint32)
        assert o == need.value
        return res

    def serial_order(self) -> np.ndarray:
        """The serialization order of the last relaxed-strategy execute (u32[n])."""
        a = np.zeros(max(self.n, 1), np.uint32)
        self._check(self.lib.gputx_read_serial_order(self.h, _ptr(a), self.n), self.h)
        return a[:self.n]

    def pool_pending(self) -> int:
        n = ctypes.c_uint64()
        self._check(self.lib.gputx_pool_pending(self.h, ctypes.byref(n)), self.h)
        return n.value

    def set_grouping(self, p: int = 0):
        """Type groups per k-set (include/gputx.h gputx_set_grouping; 0 = one per type)."""
        self._check(self.lib.gputx_set_grouping(self.h, int(p)), self.h)

    def set_chooser(self, w0_bar: int = 0, d_bar: int = 0, c_bar: int = 0):
        """Algorithm 1 thresholds for strategy "auto" (include/gputx.h gputx_set_chooser)."""
        self._check(self.lib.gputx_set_chooser(self.h, int(w0_bar), int(d_bar), int(c_bar)), self.h)

    def execute_nostats(self, strategy: str = KSET):
        self._check(self.lib.gputx_execute(self.h, STRATEGIES[strategy], None), self.h)

    def read_results(self, status: np.ndarray | None = None, out: np.ndarray | None = None, raw: bool = False):
        """(status u8[n], outputs).  Outputs: u8[n, stride]; with packed_out the packed bytes
        are read (gputx_read_results) and, unless raw, placed back at stride positions."""
        if status is None:
            status = np.zeros(self.n, np.uint8)
        if self.packed:
            off = self.read_out_offsets()
            buf = np.zeros(max(int(off[-1]), 1), np.uint8)
            self._check(self.lib.gputx_read_results(self.h, _ptr(status) if self.n else None,
                                                    _ptr(buf) if self.n else None, buf.nbytes), self.h)
            return status, (buf[:int(off[-1])] if raw else unpack_outputs(buf, off, self.stride))
        if out is None:
            out = np.zeros((self.n, self.stride), np.uint8)
        self._check(self.lib.gputx_read_results(self.h, _ptr(status) if self.n else None,
                                                _ptr(out) if self.n else None, out.nbytes), self.h)
        return status, out

    def read_out_offsets(self) -> np.ndarray:
        """gputx_read_out_offsets: u32[n + 1] byte offsets of the packed output records."""
        off = np.zeros(self.n + 1, np.uint32)
        self._check(self.lib.gputx_read_out_offsets(self.h, _ptr(off), self.n + 1, None), self.h)
        return off

    def results_device(self):
        s, o, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        self._check(self.lib.gputx_results_device(self.h, ctypes.byref(s), ctypes.byref(o), ctypes.byref(n)), self.h)
        return s.value, o.value, n.value

    def read_column(self, name: str) -> np.ndarray:
        el, cnt = self.columns[name]
        a = np.zeros(el * cnt, np.uint8)
        self._check(self.lib.gputx_read_column(self.h, name.encode(), a.ctypes.data, a.nbytes), self.h)
        return a

    def read_image(self, like: dict) -> dict:
        """All columns, viewed with the dtype/shape of `like` (e.g. the initial image)."""
        out = {}
        for name in self.columns:
            raw = self.read_column(name)
            ref = np.asarray(like[name])
            out[name] = raw.view(ref.dtype).reshape(ref.shape)
        return out

    def inserts(self) -> dict:
        res = {}
        for tab, cols in INSERT_TABLES[self.schema].items():
            rows = ctypes.c_uint64()
            self._check(self.lib.gputx_insert_rows(self.h, tab.encode(), ctypes.byref(rows)), self.h)
            res[tab] = {}
            for c in cols:
                dt = np.int32 if c in SIGNED_INSERT_COLS else np.uint32
                a = np.zeros(rows.value, dt)
                self._check(self.lib.gputx_read_insert_column(self.h, tab.encode(), c.encode(),
                                                              a.ctypes.data if a.size else None, a.nbytes), self.h)
                res[tab][c] = a
        return res

    def depths(self) -> np.ndarray:
        a = np.zeros(max(1, self.n), np.uint32)
        self._check(self.lib.gputx_read_depths(self.h, a.ctypes.data, self.n), self.h)
        return a[:self.n]

    def perm(self) -> np.ndarray:
        a = np.zeros(max(1, self.n), np.uint32)
        self._check(self.lib.gputx_read_perm(self.h, a.ctypes.data, self.n), self.h)
        return a[:self.n]

    def set_launch(self, exec_block: int = 0, exec_grid: int = 0, narrow_max: int = 0):
        self._check(self.lib.gputx_set_launch(self.h, exec_block, exec_grid, narrow_max), self.h)

    def trace_rounds(self, on: bool = True):
        self._check(self.lib.gputx_trace_rounds(self.h, int(on)), self.h)

    def round_ns(self, rounds: int) -> np.ndarray:
        """(rounds, 8) u64: CTA0 start, CTA0 signalled, CTA1 start, CTA1 signalled, polls0, polls1."""
        a = np.zeros(max(1, rounds) * 8, np.uint64)
        self._check(self.lib.gputx_read_round_ns(self.h, a.ctypes.data, rounds), self.h)
        return a[:rounds * 8].reshape(rounds, 8)

    def rank_ns(self, passes: int) -> np.ndarray:
        """(passes, 8) u64: start, A done, past bar 1, D done, past bar 2, tiles swept, sweeps."""
        a = np.zeros(max(1, passes) * 8, np.uint64)
        self._check(self.lib.gputx_read_rank_ns(self.h, a.ctypes.data, passes), self.h)
        return a[:passes * 8].reshape(passes, 8)

    def reset(self):
        self._check(self.lib.gputx_reset(self.h), self.h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.gputx_close_db(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
