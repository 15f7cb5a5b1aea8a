"""Pipelined host-resident applies: z_k = P^{-1} A x_k for a sequence of host vectors.

The reference applies its operator and preconditioner to one host vector at a
time (``_Workspace.operator(...).matvec`` + ``FastDiagPreconditioner.apply``,
solver.py:213-236, linalg.py:206-356).  When many vectors live on the host
(several right-hand sides, successive time windows, a serving queue), the
PCIe transfers dominate a serial device apply: at cfg 4 a vector is 1.5 GB
each way against ~68 ms of device work.  ``ApplyStream`` issues, per vector,

  * the host->device copy on a copy-in stream,
  * the apply (A, then optionally P^{-1}) on a compute stream,
  * the device->host copy on a copy-out stream,

with ``depth`` device buffers per side, so the copies of vectors k+1 and k-1
overlap the apply of vector k (PCIe is full duplex).  Every vector still
crosses PCIe both ways; results are bitwise identical to the serial path.
"""

import torch


class ApplyStream:
    def __init__(self, operator, precond=None, depth=2):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.op = operator
        self.pc = precond
        ctx = operator.ctx
        self.device = ctx.device
        n = operator.shape[0]
        if precond is not None and precond.shape[0] != n:
            raise ValueError("operator and preconditioner sizes differ")
        self.n = n
        self.xd = [ctx.empty(n) for _ in range(depth)]
        self.zd = [ctx.empty(n) for _ in range(depth)]
        self.yd = ctx.empty(n) if precond is not None else None
        self.s_in = torch.cuda.Stream(self.device)
        self.s_c = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)
        self.in_ready = [torch.cuda.Event() for _ in range(depth)]
        self.done = [torch.cuda.Event() for _ in range(depth)]
        self.out_done = [torch.cuda.Event() for _ in range(depth)]

    def run(self, xs, zs):
        """Issue z = P^{-1} A x (or A x without a preconditioner) for every pair
        (xs[k], zs[k]) of host fp64 tensors (pinned for overlap).  Asynchronous:
        ordered after the caller's current stream, and the caller's current
        stream is made to wait for the last copy-out before returning."""
        if len(xs) != len(zs):
            raise ValueError("xs and zs differ in length")
        for x, z in zip(xs, zs):
            if x.numel() != self.n or z.numel() != self.n:
                raise ValueError("dimension mismatch: stream of size %d" % self.n)
            if x.dtype != torch.float64 or z.dtype != torch.float64:
                raise ValueError("host vectors must be float64")
        caller = torch.cuda.current_stream(self.device)
        depth = len(self.xd)
        for s in (self.s_in, self.s_c, self.s_out):
            s.wait_stream(caller)
        for k, (xh, zh) in enumerate(zip(xs, zs)):
            b = k % depth
            with torch.cuda.stream(self.s_in):
                if k >= depth:
                    self.s_in.wait_event(self.done[b])          # apply k - depth has read xd[b]
                self.xd[b].copy_(xh.reshape(-1), non_blocking=True)
                self.in_ready[b].record(self.s_in)
            with torch.cuda.stream(self.s_c):
                self.s_c.wait_event(self.in_ready[b])
                if k >= depth:
                    self.s_c.wait_event(self.out_done[b])       # zd[b] of vector k - depth is out
                if self.pc is None:
                    self.op.apply_device(self.xd[b], self.zd[b])
                else:
                    self.op.apply_device(self.xd[b], self.yd)
                    self.pc.apply_device(self.yd, self.zd[b])
                self.done[b].record(self.s_c)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.done[b])
                zh.reshape(-1).copy_(self.zd[b], non_blocking=True)
                self.out_done[b].record(self.s_out)
        caller.wait_stream(self.s_out)
        caller.wait_stream(self.s_c)
        caller.wait_stream(self.s_in)
