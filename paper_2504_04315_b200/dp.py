"""Data-parallel training driver (BASELINE north_star).

Training shards the record batch contiguously over ranks; every rank scales
its records by 1/N_global (Eq. 9's 1/N over the whole batch, C-A13) so the
global gradient is the plain SUM of the per-rank gradients -- the only
exchange step of the method.  One optimisation step:

    accumulate_grads(local shard, N_global)   # Eq. 9 -> backprop -> scatter (CUDA)
    all_reduce(GRADS, SUM)                    # NCCL over NVLink/NVSwitch (world > 1)
    optimizer_step()                          # Adam + EMA (CUDA), identical on every rank
or, with zero1=True (the c5 schedule of SURVEY 8(e)):
    reduce_scatter(GRADS) -> Adam on this rank's shard -> all_gather(PARAMS) -> EMA

Every rank receives the same reduced bytes and runs the same deterministic
optimiser kernel, so the replicas stay bitwise identical (no parameter
broadcast needed after initialisation).  Queries (encode/decode/pdf/sample)
shard trivially and need no collective.

The driver is backend-agnostic: ``model`` is any object exposing
``accumulate_grads_ptrs`` / ``optimizer_step`` / ``grad_tensor`` (the CUDA
``npm.Model`` via ``NpmTrainer`` below; the CPU tests plug in an oracle-backed
stand-in to exercise the sharding and reduction logic over gloo).
"""
import torch
import torch.distributed as dist


def shard_range(n_global, rank, world):
    """Contiguous shard [start, end) of rank in a batch of n_global records;
    the first n_global % world ranks get one extra record."""
    base, rem = divmod(int(n_global), int(world))
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class NpmTrainer:
    """Adapter of the C-ABI model to the DataParallel protocol."""

    def __init__(self, model):
        from . import npm
        self.npm = npm
        self.m = model
        self._grads = None

    def accumulate(self, q, wi, target, spdf, n_global, want_stats):
        npm = self.npm
        channels = target.shape[0] if target.dim() == 2 else 1
        return npm.npm_accumulate_grads(self.m.h, q, wi[0], wi[1], wi[2], target, channels, spdf, n_global,
                                        want_stats, self.m._stream())

    def optimizer_step(self, want_stats):
        return self.npm.npm_optimizer_step(self.m.h, want_stats, self.m._stream())

    def grad_tensor(self, count=None):
        if count is not None:
            return self.m.buffer_view(self.npm.BUF_GRADS, count)
        if self._grads is None:
            self._grads = self.m.buffer_view(self.npm.BUF_GRADS)
        return self._grads

    # ZeRO-1 building blocks (include/npm.h npm_shard_range ...)
    def shard_range(self, rank, world):
        return self.npm.npm_shard_range(self.m.h, rank, world)

    def optimizer_step_shard(self, rank, world, want_stats):
        return self.npm.npm_optimizer_step_shard(self.m.h, rank, world, want_stats, self.m._stream())

    def param_tensor(self, count):
        return self.m.buffer_view(self.npm.BUF_PARAMS, count)

    def ema_update(self):
        self.npm.npm_ema_update(self.m.h, self.m._stream())


class DataParallel:
    def __init__(self, model, world=None, group=None, force_allreduce=False, native=False, zero1=False):
        """native=True (CUDA model only): the library's own NCCL communicator
        (npm_get_unique_id / npm_comm_init, id broadcast over the process
        group) exchanges GRADS inside npm_optimizer_step; otherwise the
        exchange runs here through torch.distributed.

        zero1=True: instead of allreduce + a replicated
        optimiser, reduce-scatter GRADS, Adam on this rank's 1/P shard,
        all-gather PARAMS, EMA locally on the whole replicated vector (the EMA
        is elementwise in the parameters, so it needs no exchange).  The same
        update as the allreduce schedule; each rank touches the Adam moments
        of 1/P of the parameters."""
        self.t = model if hasattr(model, "accumulate") else NpmTrainer(model)
        # rank and world are taken within `group` (the default group if None)
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.reduce = self.world > 1 or force_allreduce   # force: exercise the collective at world size 1
        self.zero1 = bool(zero1)
        if native:
            from . import npm
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            uid = [npm.npm_get_unique_id() if rank == 0 else None]
            if dist.is_initialized():
                # broadcast_object_list takes a GLOBAL source rank: group rank 0's
                src = dist.get_global_rank(group, 0) if group is not None else 0
                dist.broadcast_object_list(uid, src=src, group=group)
            npm.npm_comm_init(self.t.m.h, rank, self.world, uid[0])
            if self.zero1:
                npm.npm_set_exchange(self.t.m.h, npm.EXCHANGE_ZERO1)
            self.reduce = False
            self.zero1 = False      # the library runs the sharded schedule itself

    def allreduce_grads(self):
        if self.reduce:
            dist.all_reduce(self.t.grad_tensor(), op=dist.ReduceOp.SUM, group=self.group)

    def _gloo(self):
        return dist.get_backend(self.group) == "gloo"

    def zero1_step(self, want_stats):
        """reduce-scatter GRADS -> Adam on the own shard -> all-gather PARAMS
        -> EMA over the whole vector.  (gloo has no reduce-scatter: there the
        shard comes from an allreduce, the same sums.)"""
        b, c, ch = self.t.shard_range(self.rank, self.world)
        n = self.world * ch
        g = self.t.grad_tensor(n)
        if self._gloo():
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
        else:
            dist.reduce_scatter_tensor(g[b:b + ch], g, op=dist.ReduceOp.SUM, group=self.group)
        st = self.t.optimizer_step_shard(self.rank, self.world, want_stats)
        p = self.t.param_tensor(n)
        mine = p[b:b + ch].clone()
        if self._gloo():
            dist.all_gather(list(p.split(ch)), mine, group=self.group)
        else:
            dist.all_gather_into_tensor(p, mine, group=self.group)
        self.t.ema_update()
        if want_stats:
            v = torch.tensor([st["grad_norm_sq"], st["n_nonfinite_grad"]], dtype=torch.float64, device=g.device)
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
            st = dict(st, grad_norm_sq=v[0].item(), n_nonfinite_grad=int(v[1].item()))
        return st

    def global_count(self, n_local):
        """N_global = sum of the ranks' shard sizes (shards may be unequal,
        shard_range gives the first n % world ranks one more record)."""
        if self.world == 1 or not dist.is_initialized():
            return int(n_local)
        v = torch.tensor([int(n_local)], dtype=torch.int64, device=self.t.grad_tensor().device)
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
        return int(v.item())

    def train_step(self, q, wi, target, spdf, n_local=None, n_global=None, want_stats=False):
        """One data-parallel optimisation step on this rank's shard.
        n_global defaults to the sum of the ranks' n_local (one small
        allreduce; pass it to avoid that)."""
        if n_global is None:
            n_global = self.global_count(n_local if n_local is not None else q.n)
        st = self.t.accumulate(q, wi, target, spdf, n_global, want_stats)
        if self.zero1 and self.world > 1:
            st2 = self.zero1_step(want_stats)
        else:
            self.allreduce_grads()
            st2 = self.t.optimizer_step(want_stats)
        if not want_stats:
            return None
        st = dict(st)
        st["grad_norm_sq"] = st2["grad_norm_sq"]
        st["n_nonfinite_grad"] = st2["n_nonfinite_grad"]
        if self.world > 1:
            v = torch.tensor([st["loss_proxy"], st["n_used"], st["n_zero_target"], st["n_dropped"]],
                             dtype=torch.float64, device=self.t.grad_tensor().device)
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)
            st["loss_proxy"], st["n_used"], st["n_zero_target"], st["n_dropped"] = (
                v[0].item(), int(v[1].item()), int(v[2].item()), int(v[3].item()))
        return st

    def train_stream(self, make_slice, n_local, micro_local, want_stats=False):
        """f-3: micro-step training with one exchange per step.
        Each rank cuts its n_local records into consecutive slices of
        micro_local (make_slice(a, b) -> (q, wi, target, spdf) of local
        records [a, b)); micro-step j is one optimisation step over the union
        of every rank's slice j, N_global = the sum of the ranks' slice sizes.
        Every rank runs the same number of micro-steps (that of the largest
        shard); a rank whose shard is exhausted contributes an empty slice
        (make_slice(a, a)).  Returns the per-step stats (reduced over ranks)
        if want_stats."""
        out = []
        n_max = int(n_local)
        if self.world > 1 and dist.is_initialized():
            v = torch.tensor([n_max], dtype=torch.int64, device=self.t.grad_tensor().device)
            dist.all_reduce(v, op=dist.ReduceOp.MAX, group=self.group)
            n_max = int(v.item())
        for a0 in range(0, n_max, int(micro_local)):
            a = min(a0, int(n_local))
            b = min(a0 + int(micro_local), int(n_local))
            q, wi, target, spdf = make_slice(a, b)
            st = self.train_step(q, wi, target, spdf, n_local=b - a, want_stats=want_stats)
            if want_stats:
                out.append(st)
        return out if want_stats else None
