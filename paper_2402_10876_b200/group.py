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


# cost model of one CTA's work, in SM cycles, fitted to the BERT layers run
# alone on SM shares (scripts/group_probe.py, profiles/r2_group_probe.txt): a
# 64-row stage costs ~4.0 cycles per token when the activations arrive as
# dense TMA boxes (row-run layout) and ~5.5 on the cp.async gather; every
# 256-token unit adds its pipeline fill and (partly hidden) epilogue
CYCLES_PER_TOKEN_STAGE = {"runs": 4.0, "gather": 5.5}
CYCLES_PER_UNIT = 3000.0


def plan_cost(plan, sms: int, m: int) -> float:
    """Estimated cycles of the plan's busiest CTA on ``sms`` SMs (the C
    library's own work split, tw_plan_estimate), for plan-layout inputs."""
    from . import _native

    lib = _native.load_library()
    st = _native.ctypes.c_int64()
    un = _native.ctypes.c_int32()
    _native.check(lib.tw_plan_estimate(plan._handle, int(sms), int(m),
                                       _native.ctypes.byref(st), _native.ctypes.byref(un)))
    per = CYCLES_PER_TOKEN_STAGE["runs" if plan.uses_row_runs else "gather"]
    return per * st.value + CYCLES_PER_UNIT * un.value


def choose_budgets(plans, m: int, sms: int) -> List[int]:
    """SM shares minimising the slowest plan's estimated time: for a target
    time T each plan takes the fewest SMs that meet it; T is the smallest
    candidate for which the shares fit; spare SMs go where they help most."""
    floors = [int(p.info.n_sub) for p in plans]
    if sum(floors) > sms:
        raise InvalidInputError(f"{sum(floors)} sub-tiles do not fit on {sms} SMs side by side")
    cost = [{b: plan_cost(p, b, m) for b in range(f, sms + 1)} for p, f in zip(plans, floors)]
    cands = sorted({c for table in cost for c in table.values()})

    def need(t):
        out = []
        for table in cost:
            ok = [b for b, c in table.items() if c <= t]
            if not ok:
                return None
            out.append(min(ok))
        return out

    lo, hi = 0, len(cands) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        n = need(cands[mid])
        if n is not None and sum(n) <= sms:
            hi = mid
        else:
            lo = mid + 1
    budgets = need(cands[lo])
    spare = sms - sum(budgets)
    while spare > 0:   # the slowest plan takes the next SM (if any plan still gains)
        j = max(range(len(plans)), key=lambda i: cost[i][budgets[i]])
        if budgets[j] >= sms:
            break
        budgets[j] += 1
        spare -= 1
    return budgets


class TwPlanGroup:
    """Several :class:`TwPlan` s run as one step on disjoint SM shares.

    ``m`` is the token count the split is tuned for: the shares minimise the
    slowest plan's estimated time (:func:`choose_budgets` over the library's
    own work split); ``budgets`` overrides them."""

    def __init__(self, plans: Sequence, m: int, sms: Optional[int] = None,
                 budgets: Optional[Sequence[int]] = None):
        from .executor import _torch

        torch = _torch()
        if not plans:
            raise InvalidInputError("TwPlanGroup needs at least one plan")
        self.plans = list(plans)
        dev = self.plans[0].device
        if any(p.device != dev for p in self.plans):
            raise InvalidInputError("all plans of a group must live on one device")
        total = int(self.plans[0].info.sm_count) if sms is None else int(sms)
        if budgets is not None:
            if len(budgets) != len(self.plans) or sum(budgets) > total:
                raise InvalidInputError("budgets must give one SM count per plan within the GPU")
            self.budgets = [int(b) for b in budgets]
        elif len(self.plans) == 1:
            self.budgets = [total]
        else:
            self.budgets = choose_budgets(self.plans, m, total)
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

    def run(self, xs, outs=None, out_dtype: str = "fp32", fused: Optional[bool] = None):
        """TW products of every plan (``xs[i]`` in plan i's row layout).

        ``fused`` (default: up to 4 plans) runs all of them in ONE K1 launch
        on the caller's stream (``tw_gemm_group``: plan i's CTAs on its SM
        share), so consecutive steps chain through programmatic dependent
        launch; otherwise one launch per plan on concurrent streams.  Both
        give the sequential launches' results bit for bit."""
        if fused is None:
            fused = len(self.plans) <= 4
        if not fused:
            return self._launch("run", xs, outs, out_dtype)
        return self._run_fused(xs, outs, out_dtype)

    def _run_fused(self, xs, outs, out_dtype, tew: bool = False):
        import ctypes

        from . import _native
        from .executor import _DTYPE_CODES, _dtype_name

        n = len(self.plans)
        if len(xs) != n:
            raise InvalidInputError(f"expected {n} inputs, got {len(xs)}")
        outs = list(outs) if outs is not None else [None] * n
        m = None
        layouts, lds = [], []
        for i, (p, x) in enumerate(zip(self.plans, xs)):
            use_plan = p.uses_row_runs
            rows = p.layout_rows if (use_plan or p.split) else None
            mi, ld = p._check_x(x, rows)
            if m is None:
                m = mi
            elif mi != m:
                raise InvalidInputError("a fused group launch needs the same M for every plan")
            rows_out = p.info.n_union if tew else p.info.n_condensed
            if tew and not p.has_overlay:
                raise InvalidInputError(f"plan {i} has no overlay attached")
            outs[i] = p._out(rows_out, m, outs[i], out_dtype)
            layouts.append(_native.TW_LAYOUT_PLAN if use_plan else _native.TW_LAYOUT_NATURAL)
            lds.append(ld)
        codes = {_DTYPE_CODES[_dtype_name(o.dtype)] for o in outs}
        if len(codes) != 1:
            raise InvalidInputError("a fused group launch needs one output dtype")
        vp = ctypes.c_void_p
        handles = (vp * n)(*[p._handle.value if isinstance(p._handle, vp) else p._handle
                             for p in self.plans])
        xp = (vp * n)(*[x.data_ptr() for x in xs])
        cp = (vp * n)(*[o.data_ptr() for o in outs])
        ldx = (ctypes.c_int64 * n)(*lds)
        ldc = (ctypes.c_int64 * n)(*[o.stride(0) for o in outs])
        lay = (ctypes.c_int32 * n)(*layouts)
        lib = _native.load_library()
        code = codes.pop()
        if not tew:
            _native.check(lib.tw_gemm_group(handles, n, xp, ldx, lay, cp, ldc, m, code,
                                            _native.stream_handle()))
            return outs
        # per-plan K1 workspaces (stream-ordered caching allocator, as run_tew)
        from .executor import _torch

        torch = _torch()
        wss, sizes = [], []
        for p, o in zip(self.plans, outs):
            need = ctypes.c_uint64()
            _native.check(lib.tw_plan_tew_workspace_bytes(p._handle, m, code, ctypes.byref(need)))
            ws = torch.empty(int(need.value), dtype=torch.uint8, device=o.device) if need.value else None
            wss.append(ws)
            sizes.append(int(need.value))
        wp = (vp * n)(*[w.data_ptr() if w is not None else None for w in wss])
        wb = (ctypes.c_uint64 * n)(*sizes)
        _native.check(lib.tw_gemm_tew_group(handles, n, xp, ldx, lay, cp, ldc, wp, wb, m, code,
                                            _native.stream_handle()))
        return outs

    def run_tew(self, xs, outs=None, out_dtype: str = "fp32", fused: Optional[bool] = None):
        """TEW products of every plan (each must carry an overlay).  ``fused``
        (default: up to 4 plans): K1 of every plan in one launch, then each
        plan's K2 (``tw_gemm_tew_group``); else K1 + K2 per plan on
        concurrent streams."""
        if fused is None:
            fused = len(self.plans) <= 4
        if not fused:
            return self._launch("run_tew", xs, outs, out_dtype)
        return self._run_fused(xs, outs, out_dtype, tew=True)

    def set_budgets(self, budgets: Sequence[int]) -> None:
        """New SM shares (one per plan, each >= its sub-tile count, summing
        to at most the GPU).  Launches captured earlier keep their geometry."""
        floors = [int(p.info.n_sub) for p in self.plans]
        total = int(self.plans[0].info.sm_count)
        if len(budgets) != len(self.plans) or sum(budgets) > total or any(
                b < f for b, f in zip(budgets, floors)):
            raise InvalidInputError(f"invalid SM shares {list(budgets)} (floors {floors}, {total} SMs)")
        self.budgets = [int(b) for b in budgets]
        for p, b in zip(self.plans, self.budgets):
            p.set_sm_budget(b)

    def release(self) -> None:
        """Give every plan the whole GPU again."""
        for p in self.plans:
            p.set_sm_budget(0)


def tune_budgets(groups: Sequence["TwPlanGroup"], time_fn, moves=(8, 4, 2), rounds: int = 2):
    """Measured refinement of the cost model's SM shares (an autotuner):
    coordinate moves of ``moves`` SMs between every ordered pair of plans,
    hill-climbing from the current shares, applied to every group in
    ``groups`` (same plan structure, e.g. rotating buffer sets).  ``time_fn()``
    must return the time of the caller's step with the groups' current shares
    (it is called after every change; capture any CUDA graph inside it).
    Returns (budgets, time, {budgets: time})."""
    g0 = groups[0]
    floors = [int(p.info.n_sub) for p in g0.plans]
    n = len(floors)
    seen = {}

    def measure(b):
        key = tuple(b)
        if key not in seen:
            for g in groups:
                g.set_budgets(b)
            seen[key] = float(time_fn())
        return seen[key]

    best = list(g0.budgets)
    best_t = measure(best)
    for _ in range(rounds):
        improved = False
        for d in moves:
            for i in range(n):
                for j in range(n):
                    if i == j or best[i] - d < floors[i]:
                        continue
                    cand = list(best)
                    cand[i] -= d
                    cand[j] += d
                    t = measure(cand)
                    if t < best_t:
                        best, best_t, improved = cand, t, True
        if not improved:
            break
    for g in groups:
        g.set_budgets(best)
    return best, best_t, {k: v for k, v in seen.items()}
