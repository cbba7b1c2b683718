"""Shared helpers: drive the B200 engine and a checker side by side on the
same gradient buffers (generated on the device, copied to the host for the
checker — the FixedSource/replay pattern of test_engine.cpp:29-48)."""
import numpy as np

from oracle import oracle as O
from paper_2402_13781_b200 import sparsim as S

EXACT_FIELDS = ("t", "k_prime", "density", "eps", "m_t", "c_t", "f_t", "delta", "duplicates",
                "union_count", "adjust_moves", "adjust_skips", "cap_hits", "idle_workers")


def torch_dtype(dtype):
    import torch
    return torch.float64 if dtype == "f64" else torch.float32


def np_dtype(dtype):
    return np.float64 if dtype == "f64" else np.float32


def check_record(rec, orec, ctx="", err_rtol=1e-6):
    o = O.A.record_dict(orec)
    for f in EXACT_FIELDS:
        assert getattr(rec, f) == o[f], (ctx, f, getattr(rec, f), o[f])
    assert rec.k_rank == o["k_rank"], (ctx, rec.k_rank, o["k_rank"])
    # global_err: the reference sums ||e||^2 sequentially, the device by a tree
    assert abs(rec.global_err - o["global_err"]) <= err_rtol * max(abs(o["global_err"]), 1e-300), ctx


class Pair:
    """B200 engine (in-process workers) + checker engine on identical inputs."""

    def __init__(self, cfg_kw, dtype="f32", segments=None, stream_seed=None, static=False,
                 checker="oracle", verify_replication=True, distribution=0,
                 verify_conservation=False):
        import torch
        self.torch = torch
        self.cfg_kw = dict(cfg_kw)
        self.dtype = dtype
        self.cfg = S.SparsifierConfig(**cfg_kw)
        self.eng = S.Engine(self.cfg, S.EngineOptions(dtype=dtype, static_partitions=static,
                                                       verify_replication=verify_replication,
                                                       verify_conservation=verify_conservation))
        ocfg = O.make_config(**cfg_kw)
        if checker == "reference":
            self.chk = O.RefEngine(ocfg, O.make_options(static_partitions=int(static),
                                                        verify_conservation=1))
        else:
            self.chk = O.OracleEngine(ocfg, np_dtype(dtype), static_partitions=static)
        self.checker = checker
        n_g = cfg_kw["n_g"]
        self.spec = S.StreamSpec(n_g=n_g, segments=segments,
                                 seed=cfg_kw.get("seed", 42) if stream_seed is None else stream_seed,
                                 distribution=distribution)
        self.src = S.SyntheticStream(self.spec)
        self.n = self.cfg.n
        self.bufs = [torch.empty(n_g, dtype=torch_dtype(dtype), device="cuda") for _ in range(self.n)]

    def gradients(self, t):
        for r, b in enumerate(self.bufs):
            self.src.gradient(t, r, b, self.dtype, self.eng.stream())
        self.torch.cuda.synchronize()
        return [b.cpu().numpy() for b in self.bufs]

    def step(self, t, scale=None, quantum=None):
        host = self.gradients(t)
        if scale is not None or quantum is not None:
            for b in self.bufs:
                if scale is not None:
                    b.mul_(scale)
                if quantum is not None:  # coarse grid: many equal magnitudes (ties)
                    b.copy_(self.torch.round(b / quantum) * quantum)
            self.torch.cuda.synchronize()
            host = [b.cpu().numpy() for b in self.bufs]
        rec = self.eng.step(self.bufs)
        if self.checker == "reference":
            orec = self.chk.step([h.astype(np.float64) for h in host], capture=True)
        else:
            orec = self.chk.step(host)
        return rec, orec

    def compare_state(self, ctx="", vectors=True):
        n = self.n
        for w in range(n):
            st, ost = self.eng.state(w), self.chk.state(w)
            assert st.delta == ost.delta, (ctx, w, st.delta, ost.delta)
            assert list(st.k_t[:n]) == list(ost.k_t[:n]), ctx
            assert st.topology.parts() == ost.topology.parts(), (ctx, st.topology.parts(), ost.topology.parts())
            assert st.topology.pos() == ost.topology.pos(), ctx
            if vectors:
                x, ox = self.eng.x(w), self.chk.x(w)
                e, oe = self.eng.e(w), self.chk.e(w)
                for name, got, want in (("x", x, ox), ("e", e, oe)):
                    want = np.ascontiguousarray(want.astype(got.dtype))
                    same = got.view(np.uint8) == want.view(np.uint8)
                    assert same.all(), (ctx, w, name, int(np.sum(got != want)))

    def compare_selection(self, ctx=""):
        u = self.eng.idx_global(0).astype(np.int64)
        ou = self.chk.union()
        # partitions are contiguous and visited in partition order, so the
        # device union is already the reference's sorted, unique idx_global
        assert np.array_equal(u, ou), (ctx, len(u), len(ou))
        if self.checker == "oracle":
            for w in range(self.n):
                sel = self.eng.selection(w).astype(np.int64)
                assert np.array_equal(sel, self.chk.selection(w)), (ctx, w)
                assert np.array_equal(self.eng.block_counts(w), self.chk.block_counts(w)), (ctx, w)
