"""Preallocated batched pipeline: forward-backward + Viterbi + one
Baum-Welch M-step over a fixed-shape batch (BASELINE metric workload).

One ``run`` enqueues, on the caller's current stream:
  fork:  stream A  loghmm_forward_backward (log_alpha, log_beta, gamma,
                   per-sequence statistics)
         stream B  loghmm_viterbi (path, log_joint)      -- runs concurrently
  join:  loghmm_reduce_stats -> [optional all-reduce across ranks]
         -> loghmm_mstep (-> loghmm_student_guard for Student-t states)
No host synchronisation inside ``run``; ``fetch`` reads back the small
results (total log-likelihood, the updated model block) like a user would.

``run_from_host`` is the same step fed from pinned host memory: the batch is
cut into slices of whole sequences, slice s+1's host-to-device copy runs on
a copy stream while slices <= s are in the forward-backward / Viterbi
kernels, and the statistics reduction + M-step runs once over all slices.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native, engine
from .inference import HmmModel
from .training import TrainingConfig, apply_mstep_status, model_from_record

__all__ = ["Pipeline"]


class Pipeline:
    KERNELS_PER_RUN = 3  # fb, viterbi, fused reduce+mstep (single rank)

    def __init__(self, model: HmmModel, B: int, T: int, dtype="float32", *, outputs=True,
                 config: TrainingConfig | None = None, process_group=None):
        self.model = model
        self.B, self.T = B, T
        self.td = engine.torch_dtype(dtype)
        self.ns = model.n_streams
        self.config = config or TrainingConfig()
        self.pg = process_group
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        K = model.num_states
        self.K = K
        N = B * T
        off = np.arange(B + 1, dtype=np.int64) * T
        self.y0 = torch.empty(N, dtype=self.td, device=dev)
        self.y1 = torch.empty(N, dtype=self.td, device=dev) if self.ns == 2 else None
        self.batch = engine.Batch(self.y0, self.y1, torch.from_numpy(off).to(dev), off, self.td)
        self.dm = engine.DeviceModel.from_model(model, dev)
        self.dm_next = engine.DeviceModel.empty_like(self.dm)
        width = int(_native.lib().loghmm_stats_width(K, self.ns))
        self.fb = engine.FBOutputs(
            log_alpha=torch.empty((N, K), dtype=self.td, device=dev) if outputs else None,
            log_beta=torch.empty((N, K), dtype=self.td, device=dev) if outputs else None,
            gamma=torch.empty((N, K), dtype=self.td, device=dev),
            xi=None,
            ll=torch.empty(B, dtype=torch.float64, device=dev),
            partials=torch.empty((B, width), dtype=torch.float64, device=dev),
            flags=torch.empty((B, 2), dtype=torch.int64, device=dev),
        )
        self.vit = engine.VitOutputs(
            path=torch.empty(N, dtype=torch.int64, device=dev),
            log_joint=torch.empty(B, dtype=torch.float64, device=dev),
            back=None,
            flags=torch.zeros((B, 2), dtype=torch.int64, device=dev),
        )
        self.totals = torch.empty(width + 1, dtype=torch.float64, device=dev)
        self.status = torch.zeros(self.ns * K, dtype=torch.int32, device=dev)
        self.guard = torch.zeros(self.ns * K * engine.GUARD_STRIDE, dtype=torch.float64, device=dev)
        self.need_more = torch.zeros(1, dtype=torch.int32, device=dev)
        # per-rank second-pass sums (multi-rank split only)
        self.var_sums = torch.zeros(K, dtype=torch.float64, device=dev)
        self.guard_sums = torch.zeros(K * _native.GUARD_CANDIDATES, dtype=torch.float64, device=dev)
        self.ws_fb = engine.Workspace()
        self.ws_vit = engine.Workspace()
        self.ws_red = engine.Workspace()
        self.s_fb = torch.cuda.Stream(device=dev)
        # LOGHMM_VIT_PRIO=1: Viterbi on a high-priority stream (pending Viterbi CTAs
        # are placed before pending forward-backward CTAs when an SM slot frees)
        self.s_vit = torch.cuda.Stream(device=dev, priority=-1 if os.environ.get("LOGHMM_VIT_PRIO") == "1" else 0)
        fams = self.dm.host["em"]["family"]
        self.student_streams = sorted({s for s in range(self.ns) for j in range(K)
                                       if int(fams[s, j]) == _native.FAM["student_t"]})
        var_fams = (_native.FAM["gaussian"], _native.FAM["gamma"], _native.FAM["student_t"])
        self.var_streams = [s for s in range(self.ns)
                            if any(int(fams[s, j]) in var_fams for j in range(K))]
        self.ext_streams = [s for s in range(self.ns)
                            if any(int(fams[s, j]) >= _native.FAM["lognormal"] for j in range(K))]
        if self.ext_streams and process_group is not None:
            raise NotImplementedError("multi-rank steps support the five hot-path families only")
        self.s_copy = torch.cuda.Stream(device=dev)
        self._slices = {}
        # Launch order of the two concurrent kernels.  Viterbi first by default:
        # its grid is one partial wave, the forward-backward CTAs queued after
        # it fill the remaining SM slots.  fp64 with K <= 8 and Gaussian /
        # Poisson emissions is the exception (measured, config 2: 684 vs 778 us
        # per step): the fp64 forward-backward kernel holds two 255-register
        # CTAs per SM for 3.5 waves, and the K-lane Viterbi CTAs slot in as those
        # retire instead of halving the forward-backward occupancy from the start.
        cheap = all(int(fams[s, j]) in (_native.FAM["gaussian"], _native.FAM["poisson"])
                    for s in range(self.ns) for j in range(K))
        self.default_order = "fb_first" if (self.td == torch.float64 and K <= 8 and cheap) else "vit_first"
        # per-kernel CUDA events (recorded on the stream each kernel runs on)
        self.ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for k in ("fb", "vit")}

    @property
    def kernels_per_run(self) -> int:
        # + one variance pass per variance stream, + guard & select launches
        # per Student-t stream
        return (self.KERNELS_PER_RUN + len(self.var_streams)
                + 2 * engine.GUARD_LAUNCHES * len(self.student_streams)
                + 2 * _native.EXT_MAX_PASSES * len(self.ext_streams))

    def load(self, y) -> None:
        """Copy observations [B, T] (or [B, T, 2]) into the device batch."""
        if self.ns == 2 and isinstance(y, (tuple, list)):
            self.y0.copy_(torch.as_tensor(y[0]).reshape(-1), non_blocking=True)
            self.y1.copy_(torch.as_tensor(y[1]).reshape(-1), non_blocking=True)
            return
        y = torch.as_tensor(y)
        if self.ns == 1:
            self.y0.copy_(y.reshape(-1), non_blocking=True)
        else:
            self.y0.copy_(y[..., 0].reshape(-1), non_blocking=True)
            self.y1.copy_(y[..., 1].reshape(-1), non_blocking=True)

    def run(self, time_kernels: bool = False) -> None:
        main = torch.cuda.current_stream(self.dev)
        self.s_fb.wait_stream(main)
        self.s_vit.wait_stream(main)
        # (see default_order; LOGHMM_PIPE_ORDER = vit_first | fb_first | serial
        # overrides it, a measurement aid)
        order = os.environ.get("LOGHMM_PIPE_ORDER", self.default_order)

        def launch_vit():
            with torch.cuda.stream(self.s_vit):
                if time_kernels:
                    self.ev["vit"][0].record(self.s_vit)
                engine.viterbi(self.batch, self.dm, out=self.vit, workspace=self.ws_vit)
                if time_kernels:
                    self.ev["vit"][1].record(self.s_vit)

        def launch_fb():
            with torch.cuda.stream(self.s_fb):
                if time_kernels:
                    self.ev["fb"][0].record(self.s_fb)
                engine.forward_backward(self.batch, self.dm, stats=True, out=self.fb,
                                        workspace=self.ws_fb)
                if time_kernels:
                    self.ev["fb"][1].record(self.s_fb)
                # the statistics reduction and the M-step depend on the
                # forward-backward kernel only: they follow it on its stream and
                # overlap whatever is left of the Viterbi kernel
                self._tail()

        if order == "fb_first":
            launch_fb()
            launch_vit()
        elif order == "serial":
            launch_vit()
            self.s_fb.wait_stream(self.s_vit)
            launch_fb()
        else:
            launch_vit()
            launch_fb()
        main.wait_stream(self.s_fb)
        main.wait_stream(self.s_vit)

    def _tail(self) -> None:
        """Statistics reduction (+ all-reduce across ranks), M-step and the
        exact second passes, on the current stream."""
        if self.pg is None:
            # single rank: block reduction and M-step in one launch
            engine.reduce_mstep(self.fb.partials, self.fb.ll, self.totals, self.dm, self.B,
                                self.config, self.dm_next, self.status, self.guard, self.td,
                                workspace=self.ws_red)
        else:
            engine.reduce_mstep(self.fb.partials, self.fb.ll, self.totals, workspace=self.ws_red)
            self._all_reduce(self.totals)
            engine.mstep(self.dm, self.totals, self.B * self._world(), self.config, self.dm_next,
                         self.status, self.guard, self.td)
        # exact second passes (two-pass variance, ECME likelihood guard); with
        # a process group their data sums are all-reduced before the finish,
        # exactly like the statistics vector (sequences are sharded)
        for s in self.var_streams:
            if self.pg is None:
                engine.variance_pass(self.batch, self.dm_next, self.fb.gamma, s, self.guard,
                                     self.status)
            else:
                engine.variance_partial(self.batch, self.dm_next, self.fb.gamma, s, self.guard,
                                        self.var_sums)
                self._all_reduce(self.var_sums)
                engine.variance_finish(self.dm_next, s, self.guard, self.var_sums, self.status)
        # ECME guard (distributions.py:1080-1086): the full halving sequence,
        # in fixed candidate batches so the step needs no host round trip (a
        # batch with no pending state exits at once); training.baum_welch polls
        # need_more instead, with identical results
        for s in self.student_streams:
            for i in range(engine.GUARD_LAUNCHES):
                ncand = engine.guard_candidates(i)
                if self.pg is None:
                    engine.student_guard(self.batch, self.dm_next, self.fb.gamma, s,
                                         ncand, self.guard, self.status, self.need_more)
                else:
                    engine.student_guard_partial(self.batch, self.dm_next, self.fb.gamma, s,
                                                 ncand, self.guard, self.guard_sums)
                    self._all_reduce(self.guard_sums)
                    engine.student_guard_select(self.dm_next, s, ncand,
                                                self.guard, self.guard_sums, self.status,
                                                self.need_more)

        # families 6..15: the weighted-sample fit passes (fixed count; a pass
        # with nothing pending exits at once)
        for s in self.ext_streams:
            engine.ext_fit(self.batch, self.dm_next, self.fb.gamma, s, self.guard, self.status,
                           self.need_more, poll=False)

    def _all_reduce(self, t: torch.Tensor) -> None:
        import torch.distributed as dist

        dist.all_reduce(t, group=self.pg)

    def check(self) -> list[int]:
        """Host read of the step's per-state M-step status: raises
        TrainingError / warns FitWarning exactly as baum_welch does
        (training.py:130-148) and returns the collapsed states."""
        fams = [[int(self.dm.host["em"][s, j]["family"]) for j in range(self.K)]
                for s in range(self.ns)]
        return apply_mstep_status(self.status.cpu().numpy(), fams)

    def _slice_plan(self, n: int):
        """Per-slice views (batch, FB outputs, Viterbi outputs) of n equal
        slices of whole sequences."""
        if n in self._slices:
            return self._slices[n]
        B, T = self.B, self.T
        bounds = [B * i // n for i in range(n + 1)]
        plans = []
        for i in range(n):
            b0, b1 = bounds[i], bounds[i + 1]
            if b1 <= b0:
                continue
            r0, r1 = b0 * T, b1 * T
            off = np.arange(b1 - b0 + 1, dtype=np.int64) * T
            batch = engine.Batch(self.y0[r0:r1], self.y1[r0:r1] if self.y1 is not None else None,
                                 torch.from_numpy(off).to(self.dev), off, self.td)
            fb = engine.FBOutputs(
                log_alpha=self.fb.log_alpha[r0:r1] if self.fb.log_alpha is not None else None,
                log_beta=self.fb.log_beta[r0:r1] if self.fb.log_beta is not None else None,
                gamma=self.fb.gamma[r0:r1], xi=None, ll=self.fb.ll[b0:b1],
                partials=self.fb.partials[b0:b1], flags=self.fb.flags[b0:b1])
            vit = engine.VitOutputs(path=self.vit.path[r0:r1], log_joint=self.vit.log_joint[b0:b1],
                                    back=None, flags=self.vit.flags[b0:b1])
            plans.append((r0, r1, batch, fb, vit, torch.cuda.Event()))
        self._slices[n] = plans
        return plans

    def run_from_host(self, y_host, slices: int = 8) -> None:
        """One step whose observations come from (pinned) host memory, with
        the host-to-device copy of each slice overlapped with the kernels of
        the slices before it."""
        if self.ns == 2 and isinstance(y_host, (tuple, list)):
            # two pinned 1-D streams (a [B, T, 2] array's per-stream views are
            # strided: flattening them would stage through pageable memory)
            ys = [torch.as_tensor(y_host[0]).reshape(-1), torch.as_tensor(y_host[1]).reshape(-1)]
        else:
            y = torch.as_tensor(y_host)
            ys = [y.reshape(-1)] if self.ns == 1 else [y[..., 0].reshape(-1), y[..., 1].reshape(-1)]
        dst = [self.y0] if self.ns == 1 else [self.y0, self.y1]
        main = torch.cuda.current_stream(self.dev)
        plans = self._slice_plan(slices)
        self.s_copy.wait_stream(main)
        self.s_fb.wait_stream(main)
        self.s_vit.wait_stream(main)
        with torch.cuda.stream(self.s_copy):
            for r0, r1, _, _, _, ev in plans:
                for d, src in zip(dst, ys):
                    d[r0:r1].copy_(src[r0:r1], non_blocking=True)
                ev.record(self.s_copy)
        for _, _, batch, fb, vit, ev in plans:
            self.s_vit.wait_event(ev)
            with torch.cuda.stream(self.s_vit):
                engine.viterbi(batch, self.dm, out=vit, workspace=self.ws_vit)
            self.s_fb.wait_event(ev)
            with torch.cuda.stream(self.s_fb):
                engine.forward_backward(batch, self.dm, stats=True, out=fb, workspace=self.ws_fb)
        # reduction + M-step behind the last slice's forward-backward kernel on
        # its stream (they overlap the last slice's Viterbi kernel)
        with torch.cuda.stream(self.s_fb):
            self._tail()
        main.wait_stream(self.s_copy)
        main.wait_stream(self.s_fb)
        main.wait_stream(self.s_vit)

    def _world(self) -> int:
        import torch.distributed as dist

        return dist.get_world_size(self.pg)

    def kernel_ms(self) -> dict:
        return {k: a.elapsed_time(b) for k, (a, b) in self.ev.items()}

    def fetch(self):
        """Small device->host read of the step's result: total log-likelihood
        and the updated model."""
        total = float(self.totals[-1].item())
        rec = self.dm_next.to_host()
        return total, rec

    def updated_model(self) -> HmmModel:
        return model_from_record(self.dm_next.to_host())

    @property
    def d2h_bytes(self) -> int:
        return 8 + _native.MODEL_DTYPE.itemsize
