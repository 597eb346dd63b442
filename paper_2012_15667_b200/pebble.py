"""Exact oracles for the red-blue pebble game and S-partitions on tiny DAGs
(reference ``pkg/src/convio/pebble.py``) -- theory tooling that validates the
analytic bounds of :mod:`.bounds` empirically (Hong & Kung, PAPER §2-3).

Game rules (as in the reference):

* vertices without predecessors are inputs and hold blue pebbles from the
  start, so loading one is always legal;
* every output (no successors) must end with a blue pebble placed by an
  explicit Store -- also an output that is an input;
* Compute places a red pebble on a vertex whose predecessors are all red;
  re-computation is allowed; at most ``s`` red pebbles at any time;
* cost = number of Loads + Stores (Compute and eviction are free).

All sets are integer bitmasks internally; the DAGs are at most a few dozen
vertices (``DEFAULT_PEBBLE_CAP``, ``DEFAULT_PARTITION_CAP``).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass
from itertools import combinations

from .dag import Dag

DEFAULT_PEBBLE_CAP = 25
DEFAULT_PARTITION_CAP = 12


class PebbleCapError(ValueError):
    """The DAG is too large for an exact oracle."""


class PebbleInfeasibleError(ValueError):
    """No complete calculation exists with this many red pebbles."""


def _bitsof(mask: int):
    while mask:
        low = mask & -mask
        yield low.bit_length() - 1
        mask ^= low


def _pred_masks(dag: Dag) -> tuple[list[int], int, int]:
    pred = dag.predecessors()
    succ = dag.successors()
    pm = [sum(1 << u for u in set(pred[v])) for v in range(dag.n_vertices)]
    inputs = sum(1 << v for v in range(dag.n_vertices) if not pred[v])
    outputs = sum(1 << v for v in range(dag.n_vertices) if not succ[v])
    return pm, inputs, outputs


# ---------------------------------------------------------------------------
# minimum I/O of a complete calculation
# ---------------------------------------------------------------------------

def min_io_pebbling(dag: Dag, s: int, cap: int = DEFAULT_PEBBLE_CAP) -> int:
    """Exact minimum Load + Store count with ``s`` red pebbles.

    Shortest path (A*, admissible heuristic = outputs not yet stored) over
    states (red set, stored set).  Evictions are only generated when all ``s``
    red pebbles are placed: evicting earlier never shortens a calculation,
    since the pebble could be removed just before its slot is needed.
    """
    n = dag.n_vertices
    if n > cap:
        raise PebbleCapError(f"dag has {n} vertices, pebbling cap is {cap}")
    if s < 1:
        raise PebbleInfeasibleError("need at least one red pebble")
    pm, inputs, outputs = _pred_masks(dag)
    # every vertex an output depends on must be computable: in-degree + 1 <= s
    needed, todo = outputs, outputs
    while todo:
        v = (todo & -todo).bit_length() - 1
        todo &= todo - 1
        new = pm[v] & ~needed
        needed |= new
        todo |= new
    for v in _bitsof(needed):
        if pm[v] and pm[v].bit_count() + 1 > s:
            raise PebbleInfeasibleError(f"vertex {v} has in-degree {pm[v].bit_count()}, "
                                        f"cannot compute with s={s}")
    computed = [v for v in range(n) if pm[v]]
    storable = outputs | ~inputs          # storing a non-output input is pointless

    dist = {(0, 0): 0}
    heap = [(outputs.bit_count(), 0, 0, 0)]      # (estimate, -cost, red, blue)
    while heap:
        _, neg, red, blue = heapq.heappop(heap)
        cost = -neg
        if dist.get((red, blue)) != cost:
            continue
        if outputs & ~blue == 0:
            return cost

        def relax(r2: int, b2: int, c2: int) -> None:
            if c2 < dist.get((r2, b2), c2 + 1):
                dist[(r2, b2)] = c2
                heapq.heappush(heap, (c2 + (outputs & ~b2).bit_count(), -c2, r2, b2))

        if red.bit_count() >= s:
            for v in _bitsof(red):
                relax(red & ~(1 << v), blue, cost)
        else:
            for v in _bitsof((inputs | blue) & ~red):
                relax(red | (1 << v), blue, cost + 1)
            for v in computed:
                bit = 1 << v
                if not red & bit and pm[v] & ~red == 0:
                    relax(red | bit, blue, cost)
        for v in _bitsof(red & ~blue & storable):
            relax(red, blue | (1 << v), cost + 1)
    raise PebbleInfeasibleError(f"no complete calculation found with s={s}")


# ---------------------------------------------------------------------------
# dominators, generated and minimum sets
# ---------------------------------------------------------------------------

def partition_universe(dag: Dag) -> set[int]:
    """Vertices an S-partition must cover: every computed vertex and every output."""
    pred, succ = dag.predecessors(), dag.successors()
    return {v for v in range(dag.n_vertices) if pred[v] or not succ[v]}


def generated_set(dag: Dag, dominator: set[int]) -> set[int]:
    """Theta(D): the vertices every input-to-vertex path of which meets ``D``
    (complement of what the inputs reach while avoiding ``D``)."""
    pred = dag.predecessors()
    reach = set()
    for v in dag.topological_order():
        if v not in dominator and (not pred[v] or any(u in reach for u in pred[v])):
            reach.add(v)
    return set(range(dag.n_vertices)) - reach


def minimum_set(dag: Dag, subset: set[int]) -> set[int]:
    """The members of ``subset`` without a successor inside it."""
    succ = dag.successors()
    return {v for v in subset if not subset.intersection(succ[v])}


def min_dominator_size(dag: Dag, subset: set[int], limit: int | None = None) -> int:
    """Smallest vertex set meeting every input-to-``subset`` path.

    Menger: the minimum vertex cut between a super-source joined to all inputs
    and a super-sink joined from ``subset``, as a max flow with every vertex
    split into a unit-capacity in/out arc (augmenting BFS paths; stops once the
    flow exceeds ``limit``).
    """
    n = dag.n_vertices
    pred = dag.predecessors()
    src, snk = 2 * n, 2 * n + 1
    inf = n + 1
    res: dict[int, dict[int, int]] = {}

    def arc(a: int, b: int, c: int) -> None:
        res.setdefault(a, {}).setdefault(b, 0)
        res.setdefault(b, {}).setdefault(a, 0)
        res[a][b] += c

    for v in range(n):
        arc(2 * v, 2 * v + 1, 1)                 # v_in -> v_out: the vertex itself
        for u in pred[v]:
            arc(2 * u + 1, 2 * v, inf)
        if not pred[v]:
            arc(src, 2 * v, inf)
    for v in subset:
        arc(2 * v + 1, snk, inf)
    flow = 0
    while limit is None or flow <= limit:
        back = {src: None}
        q = [src]
        for a in q:
            if snk in back:
                break
            for b, c in res.get(a, {}).items():
                if c > 0 and b not in back:
                    back[b] = a
                    q.append(b)
        if snk not in back:
            break
        b = snk
        while back[b] is not None:
            a = back[b]
            res[a][b] -= 1
            res[b][a] += 1
            b = a
        flow += 1
    return flow


def is_dominator(dag: Dag, dominator: set[int], subset: set[int]) -> bool:
    return subset <= generated_set(dag, dominator)


def enumerate_small_dominators(dag: Dag, max_size: int):
    """Yield ``(D, Theta(D))`` for every vertex set of size 1 .. ``max_size``."""
    for k in range(1, max_size + 1):
        for combo in combinations(range(dag.n_vertices), k):
            dom = set(combo)
            yield dom, generated_set(dag, dom)


# ---------------------------------------------------------------------------
# S-partitions
# ---------------------------------------------------------------------------

@dataclass
class SPartition:
    """A candidate S-partition (optional explicit dominator sets)."""

    subsets: list[set[int]]
    dominators: list[set[int]] | None = None

    @property
    def h(self) -> int:
        return len(self.subsets)


@dataclass
class SPartitionCheck:
    ok: bool
    clause: str | None = None
    detail: str | None = None

    def __bool__(self) -> bool:
        return self.ok


def _fail(clause: str, detail: str) -> SPartitionCheck:
    return SPartitionCheck(False, clause, detail)


def verify_s_partition(dag: Dag, partition: SPartition, s: int) -> SPartitionCheck:
    """Properties 1-4 of an S-partition (Hong & Kung): disjoint cover of the
    universe; a dominator of size <= s per subset (re-derived unless given);
    minimum set of size <= s; acyclic dependence between subsets."""
    covered: set[int] = set()
    for i, sub in enumerate(partition.subsets):
        if covered & sub:
            return _fail("property 1", f"subset {i} overlaps another")
        covered |= sub
    missing = partition_universe(dag) - covered
    if missing:
        return _fail("property 1", f"vertices {sorted(missing)} not covered")
    for i, sub in enumerate(partition.subsets):
        if not sub:
            return _fail("property 1", f"subset {i} is empty")
        if partition.dominators is None:
            if min_dominator_size(dag, sub, limit=s) > s:
                return _fail("property 2", f"no dominator of size <= {s} for subset {i}")
        else:
            dom = partition.dominators[i]
            if len(dom) > s:
                return _fail("property 2", f"|D_{i}| = {len(dom)} > {s}")
            if not is_dominator(dag, dom, sub):
                return _fail("property 2", f"D_{i} does not dominate subset {i}")
        if len(minimum_set(dag, sub)) > s:
            return _fail("property 3", f"|M_{i}| > {s}")
    # property 4: the subset-level dependence graph is acyclic
    home = {v: i for i, sub in enumerate(partition.subsets) for v in sub}
    succ = dag.successors()
    deps = [set() for _ in partition.subsets]
    for v, i in home.items():
        deps[i].update(home[w] for w in succ[v] if w in home and home[w] != i)
    color = [0] * partition.h             # 0 new, 1 on stack, 2 done
    for root in range(partition.h):
        if color[root]:
            continue
        stack = [(root, iter(deps[root]))]
        color[root] = 1
        while stack:
            i, it = stack[-1]
            j = next(it, None)
            if j is None:
                color[i] = 2
                stack.pop()
            elif color[j] == 1:
                return _fail("property 4", f"cyclic dependence through subset {root}")
            elif color[j] == 0:
                color[j] = 1
                stack.append((j, iter(deps[j])))
    return SPartitionCheck(True)


def s_partition_oracle(dag: Dag, s: int, cap: int = DEFAULT_PARTITION_CAP) -> tuple[int, SPartition]:
    """Exact P(S), the fewest subsets of any S-partition, with a witness.

    Subsets are peeled off in dependence order -- each new subset's members
    have all their predecessors already assigned or inside it -- which
    enumerates exactly the partitions with acyclic dependence; branch and
    bound on the best count found so far.
    """
    universe = sorted(partition_universe(dag))
    m = len(universe)
    if m > cap:
        raise PebbleCapError(f"{m} partitionable vertices, cap is {cap}")
    if m == 0:
        return 0, SPartition([])
    pos = {v: i for i, v in enumerate(universe)}
    pred, succ = dag.predecessors(), dag.successors()
    pmask = [sum(1 << pos[u] for u in pred[v] if u in pos) for v in universe]
    smask = [sum(1 << pos[w] for w in succ[v] if w in pos) for v in universe]
    everything = (1 << m) - 1
    memo: dict[int, bool] = {}

    def admissible(t: int) -> bool:
        ok = memo.get(t)
        if ok is None:
            ok = sum(1 for i in _bitsof(t) if not smask[i] & t) <= s and \
                min_dominator_size(dag, {universe[i] for i in _bitsof(t)}, limit=s) <= s
            memo[t] = ok
        return ok

    best: list = [m + 1, []]

    def grow(done: int, chosen: list[int]) -> None:
        if done == everything:
            if len(chosen) < best[0]:
                best[0], best[1] = len(chosen), list(chosen)
            return
        if len(chosen) + 1 >= best[0]:
            return
        left = everything & ~done
        t = left
        while t:                           # every non-empty subset of the rest, largest first
            if all(pmask[i] & ~(done | t) == 0 for i in _bitsof(t)) and admissible(t):
                chosen.append(t)
                grow(done | t, chosen)
                chosen.pop()
                if len(chosen) + 1 >= best[0]:
                    return
            t = (t - 1) & left
    grow(0, [])
    if best[0] > m:
        raise PebbleInfeasibleError(f"no valid S-partition with s={s}")
    return best[0], SPartition([{universe[i] for i in _bitsof(t)} for t in best[1]])


def brute_force_p(dag: Dag, s: int, cap: int = DEFAULT_PARTITION_CAP) -> int:
    """P(S): the minimum number of subsets over all S-partitions."""
    return s_partition_oracle(dag, s, cap)[0]


@dataclass
class HongKungResult:
    q_min: int
    p_2s: int
    holds: bool


def check_hong_kung(dag: Dag, s: int, pebble_cap: int = DEFAULT_PEBBLE_CAP,
                    partition_cap: int = DEFAULT_PARTITION_CAP) -> HongKungResult:
    """Both exact oracles on one DAG: does ``Q >= S * (P(2S) - 1)`` hold?"""
    q = min_io_pebbling(dag, s, cap=pebble_cap)
    p2 = brute_force_p(dag, 2 * s, cap=partition_cap)
    return HongKungResult(q, p2, q >= s * (p2 - 1))
