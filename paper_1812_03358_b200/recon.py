"""PWLS reconstruction driver (paper §5, Appendix A) over the C ABI: orchestration only.

Per FISTA iteration (reading Z18; tab,alg P:349 is missing):
  1. Ax_c = A_c z               (lfm_A_forward, every camera of this rank; with ordered subsets
                                 (sec,subset) the subset prediction lfm_A_forward_subset instead)
  2. s_c = [y'WAx, y'Wy, Ax'WAx] (lfm_pwls_stats)  -> all-reduce over ranks (multi-GPU)
  3. gamma = gains(s)           (lfm_pwls_gains, on device; gamma_1 = 1)
  4. grad = sum_c A_c^T W_c (A_c z - gamma_c y_c) (+ grad R + nu on rank 0)  (lfm_pwls_grad)
     -> all-reduce grad over ranks (multi-GPU)
  5. x, z updated in place      (lfm_fista_update); t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2 on the host
The majoriser d = sum_c A_c^T W_c A_c 1 + 36 beta is computed once (lfm_majoriser).

concurrent=True (default with several cameras on one rank): steps 1-2 and each camera's backprojection in step 4
run on one CUDA stream and workspace per camera (the cameras' kernels fill each other's tails, as in bench.py's
pair); camera c > first backprojects into a private volume, the volumes are summed into grad in camera order
(lfm_vol_accumulate) and the regulariser is added last (lfm_pwls_grad with LFM_GRAD_ACCUMULATE) -- the same
additions in the same order as the sequential call.
"""
import math

import torch

from . import lfm


class PWLS:
    def __init__(self, plan, ys, ws, beta, nu=0.0, path=lfm.COLLAPSED, cams=None, group=None, concurrent=True):
        """ys, ws: per-camera device tensors (None for cameras not on this rank); cams: this rank's camera range."""
        self.plan = plan
        self.ys, self.wts = ys, ws
        self.beta, self.nu, self.path = beta, nu, path
        self.cam0, self.cam1 = cams if cams is not None else (0, plan.n_cam)
        self.group = group
        self.rank0 = group is None or torch.distributed.get_rank(group) == 0
        inf = plan.infos[0]
        dev = "cuda:%d" % plan.device
        self.n_vox = inf["n_vox"]
        self.ws = plan.workspace()
        self.Ax = [torch.empty(plan.infos[c]["n_pix"], device=dev) if self.cam0 <= c < self.cam1 else None
                   for c in range(plan.n_cam)]
        self.stats = torch.zeros(plan.n_cam * 3, dtype=torch.float64, device=dev)
        self.gamma = torch.zeros(plan.n_cam, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.grad = torch.empty(self.n_vox, device=dev)
        self.cost = torch.zeros(2, dtype=torch.float64, device=dev)
        self.d = torch.empty(self.n_vox, device=dev)
        cams_ = list(range(self.cam0, self.cam1))
        self.concurrent = concurrent and len(cams_) > 1
        if self.concurrent:   # one stream + workspace per camera, private volumes for cameras after the first
            self.streams = {c: torch.cuda.Stream(device=dev) for c in cams_}
            self.wss = {c: (self.ws if c == cams_[0] else plan.workspace()) for c in cams_}
            self.priv = {c: torch.empty(self.n_vox, device=dev) for c in cams_[1:]}

    def _allreduce(self, t):
        if self.group is not None:
            torch.distributed.all_reduce(t, group=self.group)

    def majoriser(self):
        lfm.majoriser(self.plan, self.wts, self.beta, self.d, self.ws, self.cam0, self.cam1, mode=lfm.MAJ_SUM,
                      path=self.path)
        self._allreduce(self.d)
        lfm.majoriser(self.plan, self.wts, self.beta, self.d, self.ws, 0, 0, mode=lfm.MAJ_FINISH, path=self.path)
        return self.d

    def _gradient_concurrent(self, x, subset):
        main = torch.cuda.current_stream()
        cams_ = list(range(self.cam0, self.cam1))
        self.stats.zero_()
        for c in cams_:
            s = self.streams[c]
            s.wait_stream(main)
            with torch.cuda.stream(s):
                if subset < 0:
                    lfm.A_forward(self.plan, c, x, self.Ax[c], self.wss[c], path=self.path)
                else:
                    lfm.A_forward_subset(self.plan, c, subset, x, self.Ax[c], self.wss[c])
                lfm.pwls_stats(self.plan, c, self.Ax[c], self.ys[c], self.wts[c], self.stats[3 * c:3 * c + 3],
                               self.wss[c])
        for c in cams_:
            main.wait_stream(self.streams[c])
        self._allreduce(self.stats)
        lfm.pwls_gains(self.plan, self.stats, self.gamma, self.flag)
        for c in cams_:
            s = self.streams[c]
            s.wait_stream(main)
            with torch.cuda.stream(s):
                lfm.pwls_grad(self.plan, x, self.ys, self.wts, self.Ax, self.gamma, self.beta, self.nu,
                              self.grad if c == cams_[0] else self.priv[c], self.wss[c], c, c + 1, include_reg=False,
                              path=self.path, subset=subset)
        for c in cams_:
            main.wait_stream(self.streams[c])
        for c in cams_[1:]:
            lfm.vol_accumulate(self.priv[c], self.grad)
        if self.rank0:   # the regulariser added last, as the one-call gradient does
            lfm.pwls_grad(self.plan, x, self.ys, self.wts, self.Ax, self.gamma, self.beta, self.nu, self.grad, self.ws,
                          0, 0, include_reg=1 | lfm.GRAD_ACCUMULATE, path=self.path)
        self._allreduce(self.grad)
        return self.grad

    def gradient(self, x, with_cost=False, subset=-1):
        """Exact profiled gradient (subset < 0) or the view-subset approximation eqn,subset with
        the plan's subset `subset`: prediction, gains and backprojection all over that subset (reading Z19)."""
        if self.concurrent and not with_cost:
            return self._gradient_concurrent(x, subset)
        self.stats.zero_()
        for c in range(self.cam0, self.cam1):
            if subset < 0:
                lfm.A_forward(self.plan, c, x, self.Ax[c], self.ws, path=self.path)
            else:
                lfm.A_forward_subset(self.plan, c, subset, x, self.Ax[c], self.ws)
            lfm.pwls_stats(self.plan, c, self.Ax[c], self.ys[c], self.wts[c], self.stats[3 * c:3 * c + 3], self.ws)
        self._allreduce(self.stats)
        lfm.pwls_gains(self.plan, self.stats, self.gamma, self.flag)
        lfm.pwls_grad(self.plan, x, self.ys, self.wts, self.Ax, self.gamma, self.beta, self.nu, self.grad, self.ws,
                      self.cam0, self.cam1, include_reg=self.rank0, cost=self.cost if with_cost else None,
                      path=self.path, subset=subset)
        self._allreduce(self.grad)
        if with_cost:
            self._allreduce(self.cost)
        return self.grad

    def fista(self, iters, x=None, callback=None, subsets=False):
        """FISTA (reading Z18); subsets=True: ordered subsets, iteration it uses the plan's subset
        it mod n_subsets (sec,subset P:360-388)."""
        if subsets and not self.plan.n_subsets:
            raise ValueError("the plan was built without view subsets (Plan(..., n_subsets=M))")
        d = self.majoriser()
        x = torch.zeros(self.n_vox, device=self.grad.device) if x is None else x
        z = x.clone()
        t = 1.0
        for it in range(iters):
            g = self.gradient(z, subset=it % self.plan.n_subsets if subsets else -1)
            t_new = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
            lfm.fista_update(self.plan, x, z, g, d, t, t_new)
            t = t_new
            if callback is not None:
                callback(it, x)
        if int(self.flag.item()) != 0:
            raise lfm.LfmError(5, "zero-norm weighted data for a camera c >= 2")
        return x
