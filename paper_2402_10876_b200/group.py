"""Independent TW layers of one step launched side by side (a grouped step).

The reference runs tiles of ONE layer on a thread pool (executor.py:230-265);
a model step has several independent products (e.g. BERT's Q/K/V
projections, or the layers of different micro-batches).  Launched one after
another, every K1 launch pays its own pipeline fill and its last epilogue
with the GPU partly idle.  :class:`TwPlanGroup` instead gives each plan a
share of the SMs proportional to its work (``tw_plan_set_sm_budget``: the
plan's LPT split then runs over that share) and launches the plans on
concurrent streams forked from and joined back to the caller's stream, so
their start-up and tails overlap each other's steady state.  Each product
is computed by exactly the kernel it would run alone, on fewer SMs, so
results are bit-identical to the sequential launches.  The fork/join is
made of stream events and is CUDA-graph capturable.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

from .errors import InvalidInputError


def split_sms(costs: Sequence[float], floors: Sequence[int], sms: int) -> List[int]:
    """SM budgets proportional to ``costs`` (largest remainder), each at
    least its floor (a plan needs one CTA per 128-column sub-tile), summing
    to ``sms``.  Raises when the floors alone exceed ``sms``."""
    n = len(costs)
    if n == 0:
        return []
    if sum(floors) > sms:
        raise InvalidInputError(f"{sum(floors)} sub-tiles do not fit on {sms} SMs side by side")
    total = float(sum(costs)) or 1.0
    want = [sms * c / total for c in costs]
    out = [max(f, int(w)) for f, w in zip(floors, want)]
    order = sorted(range(n), key=lambda i: -(want[i] - int(want[i])))
    i = 0
    while sum(out) < sms:
        out[order[i % n]] += 1
        i += 1
    while sum(out) > sms:
        j = max((k for k in range(n) if out[k] > floors[k]), key=lambda k: out[k] - want[k])
        out[j] -= 1
    return out


class TwPlanGroup:
    """Several :class:`TwPlan` s run as one step on disjoint SM shares.

    ``m`` is the token count the split is tuned for (the cost model is the
    plans' 64-row k-steps per token plus a per-unit epilogue share, the same
    weights the per-plan owner split uses)."""

    def __init__(self, plans: Sequence, m: int, sms: Optional[int] = None):
        from .executor import _torch

        torch = _torch()
        if not plans:
            raise InvalidInputError("TwPlanGroup needs at least one plan")
        self.plans = list(plans)
        dev = self.plans[0].device
        if any(p.device != dev for p in self.plans):
            raise InvalidInputError("all plans of a group must live on one device")
        total = int(self.plans[0].info.sm_count) if sms is None else int(sms)
        units = -(-int(m) // 256)
        costs = [(int(p.info.stage_work) + 3 * int(p.info.n_sub)) * units for p in self.plans]
        floors = [int(p.info.n_sub) for p in self.plans]
        self.budgets = split_sms(costs, floors, total) if len(self.plans) > 1 else [total]
        for p, b in zip(self.plans, self.budgets):
            p.set_sm_budget(b)
        self.streams = [torch.cuda.Stream(device=dev) for _ in self.plans]

    def _launch(self, method: str, xs, outs, out_dtype):
        from .executor import _torch

        torch = _torch()
        if len(xs) != len(self.plans):
            raise InvalidInputError(f"expected {len(self.plans)} inputs, got {len(xs)}")
        outs = list(outs) if outs is not None else [None] * len(self.plans)
        cur = torch.cuda.current_stream()
        # outputs are allocated on the caller's stream (their lifetime follows it)
        for i, (p, x) in enumerate(zip(self.plans, xs)):
            if outs[i] is None:
                rows = p.info.n_union if method == "run_tew" else p.info.n_condensed
                outs[i] = p._out(rows, int(x.shape[1]), None, out_dtype)
        fork = torch.cuda.Event()
        fork.record(cur)
        joins = []
        for p, s, x, o in zip(self.plans, self.streams, xs, outs):
            s.wait_event(fork)
            o.record_stream(s)
            x.record_stream(s)
            with torch.cuda.stream(s):
                getattr(p, method)(x, out=o, stream=s)
            e = torch.cuda.Event()
            e.record(s)
            joins.append(e)
        for e in joins:
            cur.wait_event(e)
        return outs

    def run(self, xs, outs=None, out_dtype: str = "fp32"):
        """TW products of every plan (``xs[i]`` in plan i's row layout)."""
        return self._launch("run", xs, outs, out_dtype)

    def run_tew(self, xs, outs=None, out_dtype: str = "fp32"):
        """TEW products of every plan (each must carry an overlay)."""
        return self._launch("run_tew", xs, outs, out_dtype)

    def release(self) -> None:
        """Give every plan the whole GPU again."""
        for p in self.plans:
            p.set_sm_budget(0)
