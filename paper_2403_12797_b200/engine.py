"""PosteriorEngine: the fused FAGP posterior pipeline with every buffer preallocated.

One engine per (basis, N, N*) shape.  ``run`` issues, on the current CUDA stream:

    fagp_gram_x(X, y)                                  K1   eigenfunctions on chip + DMMA Gram (+ t)
    [all_reduce(SUM) of the packed Gram over `group`]  C1   NCCL over NVLink when sharded
    fagp_factor                                        K2-K4  A, Cholesky+jitter, w, predict operand
    fagp_predict_x(X*)                                 K5   eigenfunctions on chip + DMMA mean + variance

(no basis table reaches HBM on the fused shapes; the others evaluate one into the workspace)

and never waits for the host between the factor and the prediction: attempt 0 of the factor
(no jitter) is enqueued asynchronously and its breakdown status read after the step; only a
breakdown (jitter needed) re-runs the factor through the blocking schedule and the prediction.  No allocation happens inside
``run``, so it is safe to time and to call repeatedly.
"""

from __future__ import annotations

import os

import ctypes

from . import _device as dev
from . import _lib
from .errors import NumericalError
from .mercer import LAMBDA_FLOOR_REL, Basis, raise_nonfinite

JITTER_ATTEMPTS = 3  # backend.py:165
_GPU_TRACE = None  # diagnostics: a list collects [(mark, ms since entry)] per run_host call (CUDA events)
_TRACE = None  # diagnostics: set to a list to collect run_host phase times in ms (tools/e2e_probe.py)


def _parallel_copy(dst, src):
    """dst[...] = src (C-contiguous float64 arrays of the same size) through fagp_host_copy:
    threads and non-temporal stores (staging a caller's numpy inputs into pinned memory is
    memcpy-bound at ~5 GB/s on one core, and a DMA from freshly written, cache-dirty lines runs at
    about half speed)."""
    import numpy as np

    s = np.ascontiguousarray(src, dtype=np.float64)
    if s.size != dst.size:
        raise ValueError("staging copy: size mismatch")
    threads = min(8, os.cpu_count() or 1)
    _lib.check(_lib.lib().fagp_host_copy(dst.ctypes.data, s.ctypes.data, s.nbytes, threads), "host_copy")


def _free_refcount():
    """sys.getrefcount of a pool entry's ndarray that nobody else holds, measured on the same
    code path as _out_buffer's check (pool tuple + loop name + call argument): the interpreter's
    own count, not a hard-coded literal (CPython 3.14 borrows stack references)."""
    global _FREE_RC
    if _FREE_RC is None:
        import sys

        import numpy as np

        pool = [(None, np.empty(1))]
        for _t, arr in pool:
            _FREE_RC = sys.getrefcount(arr)
    return _FREE_RC


_FREE_RC = None


class PosteriorEngine:
    def __init__(self, kernel, n_eigen, N, Ns, noise_var, mean_const=0.0, delta2_variant="rho_squared",
                 device=None, group=None, want_var=True, keep_gram=False):
        L = _lib.lib()
        self.basis = Basis(kernel, n_eigen, delta2_variant, device=device)
        b = self.basis
        self.device = b.table.device
        self.N, self.Ns = int(N), int(Ns)
        self.noise_var = float(noise_var)
        self.mean_const = float(mean_const)
        self.group = group
        self.want_var = want_var
        m, W = b.m, b.width
        e = lambda *shape: dev.empty(shape, device=self.device)  # noqa: E731
        self.packed = e(int(L.fagp_gram_len(b.ref)))
        self.gram_ws_bytes = int(L.fagp_gram_x_workspace_size(self.N, b.ref))
        self.gram_ws = e(max(1, -(-self.gram_ws_bytes // 8)))
        self.pred_ws_bytes = int(L.fagp_predict_x_workspace_size(self.Ns, b.ref))
        self.pred_ws = e(max(1, -(-self.pred_ws_bytes // 8)))
        self.lam, self.lam_floored, self.sqrt_lam = e(m), e(m), e(m)
        # modal shapes factor through the block sweep (A^{-1} only, fagp_factor_inv); p = 1
        # keeps the Cholesky route (its predict operand is built from L^{-1})
        self.inverse_route = bool(L.fagp_factor_inv(None, b.ref, None, 1.0, 0, None, None, None, None, None, None,
                                                     None, None, 0, None) != _lib.FAGP_EUNSUPPORTED)
        # fused Gram shapes take the one-launch pipelined upload path in run_host (probe: the
        # shape check comes before the argument checks)
        self.pipelined_gram = bool(L.fagp_gram_x_pipelined(None, self.N, b.ref, None, 0.0, None, None, None, 0,
                                                           None, None) != _lib.FAGP_EUNSUPPORTED)
        self.L = None if self.inverse_route else e(m, m)
        self.Ainv = e(m, m) if self.inverse_route else None
        self.G = e(m, m) if keep_gram else None
        self.t, self.w = e(m), e(m)
        self.predict_op = e(int(L.fagp_predict_operand_len(b.ref)))
        self.factor_ws_bytes = int(L.fagp_factor_workspace_size(m))
        self.factor_ws = e(max(1, self.factor_ws_bytes // 8))
        self.mean = e(self.Ns)
        self.var = e(self.Ns) if want_var else None
        self.flags = dev.zeros((2,), dtype="int32", device=self.device)
        self.jitter = ctypes.c_double(0.0)
        self.pivot = ctypes.c_int32(0)
        self.status = 0
        _lib.check(L.fagp_eigenvalues(b.ref, LAMBDA_FLOOR_REL, _lib.ptr(self.lam), _lib.ptr(self.lam_floored),
                                      _lib.ptr(self.sqrt_lam), _lib.stream_handle()), "eigenvalues")

    def _flag(self, k):
        return ctypes.c_void_p(self.flags.data_ptr() + 4 * k)

    # -- stages (each usable alone, e.g. for per-kernel timing) --------------------------
    def table(self, X, y=None, flag=None):
        """The 1-D eigenfunction table of X (fagp_basis_eval): only for the error path (naming
        a non-finite feature) and the optional full covariance -- never on the hot path."""
        L, b = _lib.lib(), self.basis
        T = dev.empty((int(X.shape[0]), b.width), device=self.device)
        if X.shape[0]:
            _lib.check(L.fagp_basis_eval(_lib.ptr(X), int(X.shape[0]), b.ref, _lib.ptr(y), self.mean_const,
                                         _lib.ptr(T), flag, _lib.stream_handle()), "basis_eval")
        return T

    def stage_gram(self, X, y, stream=None):
        """K1: eigenfunctions of the train rows + Gram [K | t] (fagp_gram_x)."""
        L, s, b = _lib.lib(), _lib.stream_handle(stream), self.basis
        _lib.check(L.fagp_gram_x(_lib.ptr(X), self.N, b.ref, _lib.ptr(y), self.mean_const, _lib.ptr(self.packed),
                                 _lib.ptr(self.gram_ws), self.gram_ws_bytes, self._flag(0), s), "gram")

    def stage_reduce(self):
        if self.group is not None:
            from .distributed import all_reduce_sum

            all_reduce_sum(self.packed, self.group)

    def stage_factor(self, stream=None):
        L, s, b = _lib.lib(), _lib.stream_handle(stream), self.basis
        if self.inverse_route:
            self.status = L.fagp_factor_inv(_lib.ptr(self.packed), b.ref, _lib.ptr(self.sqrt_lam), self.noise_var,
                                            JITTER_ATTEMPTS, _lib.ptr(self.Ainv), _lib.ptr(self.G), _lib.ptr(self.t),
                                            _lib.ptr(self.w), _lib.ptr(self.predict_op), ctypes.byref(self.jitter),
                                            ctypes.byref(self.pivot), _lib.ptr(self.factor_ws), self.factor_ws_bytes,
                                            s)
            if self.status not in (_lib.FAGP_OK, _lib.FAGP_ENOTPD):
                _lib.check(self.status, "factor")
            return self.status
        self.status = L.fagp_factor(_lib.ptr(self.packed), b.ref, _lib.ptr(self.sqrt_lam), self.noise_var,
                                    JITTER_ATTEMPTS, _lib.ptr(self.L), _lib.ptr(self.G), _lib.ptr(self.t),
                                    _lib.ptr(self.w), _lib.ptr(self.predict_op), ctypes.byref(self.jitter),
                                    ctypes.byref(self.pivot), _lib.ptr(self.factor_ws), self.factor_ws_bytes, s)
        if self.status not in (_lib.FAGP_OK, _lib.FAGP_ENOTPD):
            _lib.check(self.status, "factor")
        return self.status

    def stage_factor_async(self, stream=None):
        """Attempt 0 of the factorisation with no host synchronisation (fagp_factor_inv_async):
        the prediction can be queued right behind it.  Returns False when the shape has no
        async route (the blocking stage_factor ran instead and its status is in self.status).
        After the stream has synchronised, factor_needs_retry() says whether the breakdown path
        (jitter schedule) has to run."""
        import torch

        if not self.inverse_route:
            self.stage_factor(stream)
            return False
        L, s, b = _lib.lib(), _lib.stream_handle(stream), self.basis
        if getattr(self, "info_host", None) is None:
            self.info_host = torch.zeros((1,), dtype=torch.int32, pin_memory=True)
        self.info_host.zero_()
        rc = L.fagp_factor_inv_async(_lib.ptr(self.packed), b.ref, _lib.ptr(self.sqrt_lam), self.noise_var,
                                     _lib.ptr(self.Ainv), _lib.ptr(self.G), _lib.ptr(self.t), _lib.ptr(self.w),
                                     _lib.ptr(self.predict_op), _lib.ptr(self.info_host), _lib.ptr(self.factor_ws),
                                     self.factor_ws_bytes, s)
        _lib.check(rc, "factor")
        self.jitter.value = 0.0
        self.pivot.value = 0
        self.status = _lib.FAGP_OK
        return True

    def factor_needs_retry(self):
        """After a synchronisation: did the async attempt break down (jitter schedule needed)?"""
        return getattr(self, "info_host", None) is not None and int(self.info_host[0]) != 0

    def set_mean_weights(self, stream=None):
        _lib.check(_lib.lib().fagp_set_mean_weights(_lib.ptr(self.predict_op), _lib.ptr(self.w), self.basis.ref,
                                                    _lib.stream_handle(stream)), "set_mean_weights")

    def stage_predict(self, Xs, stream=None):
        """K5: eigenfunctions of the test rows + mean and variance (fagp_predict_x)."""
        L, s, b = _lib.lib(), _lib.stream_handle(stream), self.basis
        if self.Ns:
            _lib.check(L.fagp_predict_x(_lib.ptr(Xs), self.Ns, b.ref, _lib.ptr(self.predict_op), self.noise_var,
                                        self.mean_const, _lib.ptr(self.mean), _lib.ptr(self.var), self._flag(1),
                                        _lib.ptr(self.pred_ws), self.pred_ws_bytes, s), "predict")

    # -- the whole step -------------------------------------------------------------------
    def run(self, X, y, Xs, fault_flip=False, xs_ready=None):
        """One posterior evaluation from device-resident inputs; returns device (mean, var).

        X* is first touched by the predict kernel, so an X* upload still in flight on another
        stream (``xs_ready``: its event) overlaps the Gram contraction and the factorisation."""
        import torch

        self.flags.zero_()
        self.stage_gram(X, y)
        self.stage_reduce()
        asynchronous = self.stage_factor_async()
        if xs_ready is not None:
            torch.cuda.current_stream().wait_event(xs_ready)
        if not asynchronous and self.status != _lib.FAGP_OK:
            self.raise_errors(X, Xs, y, factor_failed=True)
        if fault_flip:
            self.w.neg_()
            self.set_mean_weights()
        self.stage_predict(Xs)
        if asynchronous:
            torch.cuda.current_stream().synchronize()
            if self.factor_needs_retry():
                self._retry_factor(X, Xs, y, fault_flip)
                self.stage_predict(Xs)
        return self.mean, self.var

    def capture(self, X, y, Xs):
        """Record one device step -- flags, Gram, asynchronous factor, predict -- as a CUDA graph
        over these buffers (replay() re-runs it with whatever X, y, X* then hold): a step of ~10
        launches becomes one graph launch, no host round trips between the kernels.  Only for the
        shapes with the asynchronous factor route and no process group (the jitter decision and
        the all-reduce stay on the host path); returns None otherwise.  After a replay the caller
        synchronises and checks factor_needs_retry() (the breakdown status is copied out by the
        graph itself)."""
        import torch

        if not self.inverse_route or self.group is not None:
            return None

        def step():
            self.flags.zero_()
            self.stage_gram(X, y)
            self.stage_factor_async()
            self.stage_predict(Xs)

        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):  # warm-up outside the capture (lazy module loading, workspaces)
            step()
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        self._graph = g
        return g

    def replay(self):
        """Launch the captured step (capture() first); returns the device (mean, var)."""
        self._graph.replay()
        return self.mean, (self.var if self.want_var else None)

    def _retry_factor(self, X, Xs, y, fault_flip):
        """The async attempt broke down: run the full jitter schedule (blocking) and re-apply the
        fault hook; raises the reference's NumericalError if even the last attempt fails."""
        st = self.stage_factor()
        if st != _lib.FAGP_OK:
            self.raise_errors(X, Xs, y, factor_failed=True)
        if fault_flip:
            self.w.neg_()
            self.set_mean_weights()

    # -- the whole step from host memory (the fagp_posterior path) -------------------------
    PREDICT_CHUNKS = int(os.environ.get("FAGP_PREDICT_CHUNKS", "6"))  # tuning knob

    def _host_buffers(self):
        import torch

        if getattr(self, "X", None) is None:
            p = self.basis.p
            self.X = dev.empty((self.N, p), device=self.device)
            self.y = dev.empty((self.N,), device=self.device)
            self.Xs = dev.empty((self.Ns, p), device=self.device)
            self.s_in = torch.cuda.Stream(device=self.device)
            self.s_out = torch.cuda.Stream(device=self.device)
            self._stage = {}
        return self.X, self.y, self.Xs

    def _staging_source(self, a, shape):
        """The C-contiguous float64 host array behind `a` when it must be staged (not a pinned
        tensor already), else None."""
        import numpy as np
        import torch

        if isinstance(a, torch.Tensor):
            if a.is_pinned() and a.dtype == torch.float64 and a.is_contiguous():
                return None
            a = a.detach().cpu().numpy()
        src = np.ascontiguousarray(np.asarray(a, dtype=np.float64)).reshape(shape)
        return src

    def _stage_buf(self, key, shape):
        import torch

        buf = self._stage.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = torch.empty(shape, dtype=torch.float64, pin_memory=True)
            self._stage[key] = buf
        return buf

    def _pinned(self, a, key, shape):
        """Host source for an async H2D copy: a pinned CPU tensor as is, anything else staged
        into an engine-owned pinned buffer (one host memcpy)."""
        import numpy as np
        import torch

        if isinstance(a, torch.Tensor) and a.is_pinned() and a.dtype == torch.float64 and a.is_contiguous():
            return a.reshape(shape)
        buf = self._stage.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = torch.empty(shape, dtype=torch.float64, pin_memory=True)
            self._stage[key] = buf
        src = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
        _parallel_copy(buf.numpy(), src.reshape(shape))
        return buf

    def run_host(self, Xh, yh, Xsh, fault_flip=False):
        """One posterior evaluation from HOST inputs to host numpy (mean, var), pipelined:

          * train rows go up in fagp_gram_x_chunks() pieces on a copy stream (sub-range k of every
            CTA's rows) and Gram chunk k starts as soon as they have landed (bitwise identical
            to one fagp_gram_x call);
          * X* goes up behind them and overlaps the Gram tail and the factorisation;
          * predict runs in row chunks, each chunk's mean/var D2H overlapping the next chunk.
        Results land in fresh pinned host memory (returned as numpy views)."""
        import time

        import torch

        trace = [time.perf_counter()] if _TRACE is not None else None
        L, b = _lib.lib(), self.basis
        cs = torch.cuda.current_stream(self.device)
        gev = [] if _GPU_TRACE is not None else None

        def mark(name, stream):
            if gev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                gev.append((name, e))

        mark("start", cs)
        self._host_flags = None
        X, y, Xs = self._host_buffers()
        p = b.p
        # pageable (numpy) train inputs are staged chunk by chunk right before each chunk's upload
        # (fagp_gram_x_stage_chunk), so staging chunk k overlaps the DMA of chunk k - 1 and the
        # Gram on the chunks already landed; pinned tensors go up as they are
        x_src, y_src = self._staging_source(Xh, (self.N, p)), self._staging_source(yh, (self.N,))
        staged = x_src is not None and y_src is not None
        if staged:
            Xh, yh = self._stage_buf("X", (self.N, p)), self._stage_buf("y", (self.N,))
        else:
            Xh = self._pinned(Xh, "X", (self.N, p))
            yh = self._pinned(yh, "y", (self.N,))
        Xsh_src = Xsh  # staged (when not pinned already) once the Gram is queued: overlaps it
        threads = min(8, os.cpu_count() or 1)

        def stage(k):
            if staged:
                _lib.check(L.fagp_gram_x_stage_chunk(x_src.ctypes.data, y_src.ctypes.data, self.N, b.ref, k,
                                                     _lib.ptr(Xh), _lib.ptr(yh), threads), "stage")
        self.flags.zero_()
        nch = int(L.fagp_gram_x_chunks(self.N, b.ref))
        ready = self._ready_words(nch)
        # re-arm the ready words on the compute stream behind everything the copy stream has
        # queued so far: a late signal of an earlier call (one that timed out with STALLED)
        # lands before the zeroing, never after it
        cs.wait_stream(self.s_in)
        ready.zero_()
        self.s_in.wait_stream(cs)
        sin = _lib.stream_handle(self.s_in)
        # zero-copy train rows: pinned (mapped) X / y are read by the Gram kernel itself across
        # PCIe as it contracts (bitwise the device-resident launch), no upload chunks or ready words
        zc_in = (self.ZERO_COPY_IN and self.pipelined_gram and not staged and self._mapped(Xh)
                 and self._mapped(yh))
        if zc_in:
            _lib.check(L.fagp_gram_x(_lib.ptr(Xh), self.N, b.ref, _lib.ptr(yh), self.mean_const, _lib.ptr(self.packed),
                                     _lib.ptr(self.gram_ws), self.gram_ws_bytes, self._flag(0),
                                     _lib.stream_handle(cs)), "gram")
            mark("gram", cs)
            X, y = Xh, yh  # (error reports and retries read the rows where they are)
        elif self.pipelined_gram:
            # the copy stream uploads chunk k and then sets ready word k (a stream-ordered 4-byte
            # H2D copy); ONE Gram launch waits on the words chunk by chunk.  The copies are
            # queued first, so nothing the host does after the launch can hold them back.
            # (staged inputs: chunk 0 goes up first, then the Gram is launched, then chunks 1.. are
            # staged and uploaded while it contracts -- the launch waits on the ready words)
            def upload(k):
                stage(k)
                _lib.check(L.fagp_gram_x_upload_chunk(_lib.ptr(Xh), _lib.ptr(yh), self.N, b.ref, k, _lib.ptr(X),
                                                      _lib.ptr(y), sin), "upload")
                _lib.check(L.fagp_gram_x_signal(_lib.ptr(ready), k, sin), "signal")
                mark(f"up{k}", self.s_in)

            first = 1 if staged else nch
            for k in range(first):
                upload(k)
            _lib.check(L.fagp_gram_x_pipelined(_lib.ptr(X), self.N, b.ref, _lib.ptr(y), self.mean_const,
                                               _lib.ptr(ready), _lib.ptr(self.packed), _lib.ptr(self.gram_ws),
                                               self.gram_ws_bytes, self._flag(0), _lib.stream_handle(cs)), "gram")
            mark("gram", cs)
            for k in range(first, nch):
                upload(k)
        else:  # table-path shapes: chunk launches behind events
            for k in range(nch):
                stage(k)
                _lib.check(L.fagp_gram_x_upload_chunk(_lib.ptr(Xh), _lib.ptr(yh), self.N, b.ref, k, _lib.ptr(X),
                                                      _lib.ptr(y), sin), "upload")
                ev = torch.cuda.Event()
                ev.record(self.s_in)
                mark(f"up{k}", self.s_in)
                cs.wait_event(ev)
                _lib.check(L.fagp_gram_x_chunk(_lib.ptr(X), self.N, b.ref, _lib.ptr(y), self.mean_const, k,
                                               _lib.ptr(self.packed), _lib.ptr(self.gram_ws), self.gram_ws_bytes,
                                               self._flag(0), _lib.stream_handle(cs)), "gram")
                mark(f"gram{k}", cs)
        xs_src = self._staging_source(Xsh_src, (self.Ns, p))

        xs_read = Xs  # what the predict reads: the device copy, or a mapped pinned X* itself

        def upload_xs():
            nonlocal xs_read
            xs_host = self._pinned(Xsh_src, "Xs", (self.Ns, p))
            with torch.cuda.stream(self.s_in):
                if self.Ns and zc_in and self._mapped(xs_host):
                    xs_read = xs_host  # zero-copy: the predict loads its rows across PCIe
                elif self.Ns:
                    Xs.copy_(xs_host, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_in)
            mark("xs_up", self.s_in)
            return ev

        # a pinned X* goes up right behind the train rows; a pageable one is staged on the host
        # after the factorisation is queued (the staging then overlaps the Gram tail and factor)
        ev_xs = upload_xs() if xs_src is None else None
        Xs = xs_read
        if trace is not None:
            trace.append(time.perf_counter())
        self.stage_reduce()
        asynchronous = self.stage_factor_async()
        mark("factor", cs)
        if ev_xs is None:
            # pageable X*: staged and uploaded per predict chunk (below), chunk k + 1's host copy
            # overlapping chunk k's predict
            xs_stage = self._stage_buf("Xs", (self.Ns, p))
            ev_xs = torch.cuda.Event()
            ev_xs.record(cs)  # (nothing to wait for before the first chunk's own upload)
        else:
            xs_stage = None
        if trace is not None:
            trace.append(time.perf_counter())
        cs.wait_event(ev_xs)
        if not asynchronous and self.status != _lib.FAGP_OK:
            self.raise_errors(X, Xs, y, factor_failed=True)
        if fault_flip:
            self.w.neg_()
            self.set_mean_weights()
        rows = 2 if self.want_var else 1
        out, o = self._out_buffer(rows)
        # zero-copy results: the predict kernels store mean / var straight into the pinned result
        # buffer (mapped under unified addressing), so no D2H copy trails the last chunk and, with
        # a pinned X*, no chunking is needed at all
        zc = self.ZERO_COPY_OUT and self._mapped(out)
        chunks = self._predict_chunks() if (not zc or xs_stage is not None) else [(0, self.Ns)]
        if trace is not None:
            trace.append(time.perf_counter())
        for ci, (a, e) in enumerate(chunks):
            if xs_stage is not None and e > a:
                _parallel_copy(xs_stage[a:e].numpy(), xs_src[a:e])
                with torch.cuda.stream(self.s_in):
                    Xs[a:e].copy_(xs_stage[a:e], non_blocking=True)
                    evc = torch.cuda.Event()
                    evc.record(self.s_in)
                mark(f"xs{ci}", self.s_in)
                cs.wait_event(evc)
            dm = out[0, a:e] if zc else self.mean[a:e]
            dv = (out[1, a:e] if zc else self.var[a:e]) if self.want_var else None
            _lib.check(L.fagp_predict_x(_lib.ptr(Xs[a:e]), e - a, b.ref, _lib.ptr(self.predict_op), self.noise_var,
                                        self.mean_const, _lib.ptr(dm), _lib.ptr(dv), self._flag(1),
                                        _lib.ptr(self.pred_ws), self.pred_ws_bytes, _lib.stream_handle(cs)),
                       "predict")
            ev = torch.cuda.Event()
            ev.record(cs)
            mark(f"pred{ci}", cs)
            if zc:
                continue
            self.s_out.wait_event(ev)
            with torch.cuda.stream(self.s_out):
                out[0, a:e].copy_(self.mean[a:e], non_blocking=True)
                if self.want_var:
                    out[1, a:e].copy_(self.var[a:e], non_blocking=True)
            mark(f"d2h{ci}", self.s_out)
        if trace is not None:
            trace.append(time.perf_counter())
        # the flag words ride home with the results (no separate D2H + sync in check())
        fh = self.__dict__.get("_flags_pinned")
        if fh is None:
            fh = self._flags_pinned = torch.empty((2,), dtype=torch.int32, pin_memory=True)
        self.s_out.wait_stream(cs)
        with torch.cuda.stream(self.s_out):
            fh.copy_(self.flags, non_blocking=True)
        self.s_out.synchronize()
        self._host_flags = (int(fh[0]), int(fh[1]))
        if gev is not None:
            _GPU_TRACE.append([(n, gev[0][1].elapsed_time(e)) for n, e in gev])
        if trace is not None:
            trace.append(time.perf_counter())
            _TRACE.append([1e3 * (b - a) for a, b in zip(trace, trace[1:])])
        if asynchronous and self.factor_needs_retry():
            self._host_flags = None
            self._retry_factor(X, Xs, y, fault_flip)
            self.stage_predict(Xs)
            torch.cuda.current_stream(self.device).synchronize()
            out[0].copy_(self.mean)
            if self.want_var:
                out[1].copy_(self.var)
        return o[0], (o[1] if self.want_var else None)

    ZERO_COPY_OUT = True  # predict into the pinned result buffer when the device can map it
    ZERO_COPY_IN = True  # Gram / predict read pinned (mapped) X, y, X* in place (fused routes)

    def _mapped(self, out):
        """Whether a pinned host tensor is device-accessible at its own address (cached)."""
        key = (out.data_ptr(), out.numel())
        cache = self.__dict__.setdefault("_mapped_cache", {})
        if key not in cache:
            cache[key] = bool(_lib.lib().fagp_host_mapped(out.data_ptr(), out.numel() * out.element_size()))
        return cache[key]

    def _predict_chunks(self):
        """Row ranges of the chunked predict, cut at whole waves of the fused predict (every chunk
        but the last fills all SMs to the end; else multiples of 64 rows).  Each chunk's D2H
        overlaps the next chunk's compute, so only the last chunk's D2H is exposed: the chunks
        shrink geometrically towards the end (..., 8, 4, 2, 1 waves), the rest split evenly."""
        Ns, pc = self.Ns, max(1, self.PREDICT_CHUNKS)
        wave = int(_lib.lib().fagp_predict_x_wave_rows(self.basis.ref)) or 64
        nw = -(-max(Ns, 1) // wave)
        tail = []
        while len(tail) < pc - 2 and sum(tail) + 2 ** len(tail) <= nw // 2:
            tail.append(2 ** len(tail))
        head = nw - sum(tail)
        nh = max(1, pc - len(tail))
        sizes = [head * (i + 1) // nh - head * i // nh for i in range(nh)] + tail[::-1]
        cuts, a = [0], 0
        for w in sizes:
            a += w
            cuts.append(min(Ns, a * wave))
        return [(x, y) for x, y in zip(cuts, cuts[1:]) if y > x]

    def _ready_words(self, n):
        """Zeroed device words for fagp_gram_x_pipelined (re-armed by the launch itself)."""
        r = getattr(self, "_ready", None)
        if r is None or r.numel() != n:
            r = self._ready = dev.zeros((n,), dtype="int32", device=self.device)
        return r

    def _out_buffer(self, rows):
        """A pinned (rows, N*) result buffer no caller still holds: the returned mean/var are
        views of the pool entry's ndarray, so its refcount says whether it is free.  Avoids a
        cudaHostAlloc (milliseconds) whenever the host caching allocator misses."""
        import sys

        import torch

        pool = self.__dict__.setdefault("_out_pool", [])
        free = _free_refcount()
        for t, arr in pool:
            if arr.shape == (rows, self.Ns) and sys.getrefcount(arr) <= free:
                return t, arr
        # two at a time: the common `r = fagp_posterior(...)` loop holds one result while the
        # next call fills the other
        for _ in range(1 if pool else 2):
            t = torch.empty((rows, self.Ns), dtype=torch.float64, pin_memory=True)
            pool.append((t, t.numpy()))
        while len(pool) > 4:  # forget the oldest (views still held keep their memory alive)
            pool.pop(0)
        return pool[-1]

    def raise_errors(self, X=None, Xs=None, y=None, factor_failed=False, after_predict=False):
        """Raise the reference's exception for whatever went wrong (validation order of
        fagp_posterior: train X, train Phi, test X, test Phi, then the factorisation)."""
        hf, self._host_flags = self.__dict__.get("_host_flags"), None
        fl = list(hf) if hf is not None else [int(v) for v in dev.to_host(self.flags)]
        b = self.basis
        if fl[0] & _lib.FLAG_STALLED:
            raise RuntimeError("pipelined Gram: an input chunk was never signalled (FAGP_FLAG_STALLED)")
        if fl[0] & _lib.FLAG_X_NONFINITE:
            raise ValueError("X must be finite")
        if fl[0] & _lib.FLAG_PHI_NONFINITE:
            raise_nonfinite(self.table(X, y), X, b)
        if fl[1] & _lib.FLAG_X_NONFINITE:
            raise ValueError("X must be finite")
        if factor_failed and self.Ns and not fl[1]:
            # the test rows were not evaluated yet: do it now (sets the X* flag when needed)
            Ts = self.table(Xs, flag=self._flag(1))
            if int(dev.to_host(self.flags)[1]) & _lib.FLAG_X_NONFINITE:
                raise ValueError("X must be finite")
            raise_nonfinite(Ts, Xs, b)
        elif fl[1] & _lib.FLAG_PHI_NONFINITE and self.Ns:
            raise_nonfinite(self.table(Xs), Xs, b)
        if factor_failed:
            piv = int(self.pivot.value)
            raise NumericalError(
                f"matrix of order {b.m} is not positive definite: leading minor {piv} failed even with "
                f"diagonal jitter up to the third escalation", pivot_index=piv)

    def check(self, X, Xs, y=None):
        """Post-run validation (one small D2H read of the flag words)."""
        self.raise_errors(X, Xs, y)
