"""Computation DAGs of direct and Winograd convolution (reference ``pkg/src/convio/dag.py``).

Two layers live here:

* the closed-form lemma counts ``|V|`` the composite lower bounds consume
  (``dag.py:184-204``, used at ``bounds.py:234,256``) and the Winograd output
  padding (``dag.py:291-299``) -- the hot path;
* the materialised DAGs themselves (``Dag``, ``build_direct_conv_dag``,
  ``build_winograd_dag``, the adjacency text format and the multi-step
  partition check, ``dag.py:36-178,247-457``) -- the theory tooling the
  pebble-game oracles (:mod:`.pebble`) and the reference's soundness tests
  run on tiny graphs.  Its vertex numbering is the reference's (inputs in
  ``img[b,c,y,x]`` then ``wt[oc,c,ky,kx]`` order, then one (output pixel,
  output channel) group at a time), so an exported ``.dag`` file is
  interchangeable with one the reference writes.

Arithmetic structure (the DAG semantics every kernel and the oracle follow):
sums are left-deep chains of 2-input vertices; a linear-combination tree
first scales each leaf (one unary vertex per leaf) and then sums the scaled
values.  Transform coefficients are edge annotations and add no vertices.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

from .model import ConvShape, GeometryError, WinogradParams

# vertex kinds (reference integer codes, dag.py:16)
INPUT, INTERNAL, OUTPUT = 0, 1, 2
KIND_NAMES = {INPUT: "input", INTERNAL: "internal", OUTPUT: "output"}
KIND_IDS = {name: kind for kind, name in KIND_NAMES.items()}

DEFAULT_VERTEX_CAP = 10_000_000
_HEADER = "# convio dag v1"


class SizeCapError(ValueError):
    """Materialising the DAG would exceed the vertex cap."""


class MultiStepViolation(ValueError):
    """A clause of the multi-step partition definition fails at ``vertex``."""

    def __init__(self, vertex: int, clause: str):
        super().__init__(f"vertex {vertex}: {clause}")
        self.vertex = vertex
        self.clause = clause


# ---------------------------------------------------------------------------
# the graph
# ---------------------------------------------------------------------------

class Dag:
    """Append-only vertex/edge lists; adjacency views are built on demand."""

    def __init__(self):
        self.kinds: list[int] = []
        self.steps: list[int] = []
        self.edges: list[tuple[int, int]] = []
        self._adj: tuple[list[list[int]], list[list[int]]] | None = None

    # construction
    def add_vertex(self, kind: int, step: int = 0) -> int:
        self.kinds.append(kind)
        self.steps.append(step)
        self._adj = None
        return len(self.kinds) - 1

    def add_edge(self, src: int, dst: int) -> None:
        self.edges.append((src, dst))
        self._adj = None

    # views
    @property
    def n_vertices(self) -> int:
        return len(self.kinds)

    def _adjacency(self) -> tuple[list[list[int]], list[list[int]]]:
        if self._adj is None:
            n = self.n_vertices
            pred: list[list[int]] = [[] for _ in range(n)]
            succ: list[list[int]] = [[] for _ in range(n)]
            for a, b in self.edges:
                succ[a].append(b)
                pred[b].append(a)
            self._adj = (pred, succ)
        return self._adj

    def predecessors(self) -> list[list[int]]:
        return self._adjacency()[0]

    def successors(self) -> list[list[int]]:
        return self._adjacency()[1]

    def input_vertices(self) -> list[int]:
        return [v for v, kind in enumerate(self.kinds) if kind == INPUT]

    def output_vertices(self) -> list[int]:
        return [v for v, kind in enumerate(self.kinds) if kind == OUTPUT]

    def count_vertices(self, kinds: set[int]) -> int:
        """Number of vertices whose kind is in ``kinds``."""
        return sum(kind in kinds for kind in self.kinds) if kinds else 0

    def topological_order(self) -> list[int]:
        """A topological order (Kahn); ``ValueError`` on a cycle."""
        pred, succ = self._adjacency()
        missing = [len(p) for p in pred]
        ready = deque(v for v in range(self.n_vertices) if missing[v] == 0)
        order: list[int] = []
        while ready:
            v = ready.popleft()
            order.append(v)
            for w in succ[v]:
                missing[w] -= 1
                if missing[w] == 0:
                    ready.append(w)
        if len(order) < self.n_vertices:
            raise ValueError("dag contains a cycle")
        return order

    def step_output_sets(self) -> dict[int, set[int]]:
        """Per step label j > 0: the vertices of step j with no step-j successor
        (the outputs of sub-DAG G_j)."""
        succ = self.successors()
        out: dict[int, set[int]] = {}
        for v, j in enumerate(self.steps):
            if j and all(self.steps[w] != j for w in succ[v]):
                out.setdefault(j, set()).add(v)
        return out

    # adjacency text format (reference dag.py:119-165)
    def to_adjacency_text(self) -> str:
        head = [_HEADER, f"# vertices {self.n_vertices}"]
        head += [f"# vertex {v} {KIND_NAMES[kind]} {step}"
                 for v, (kind, step) in enumerate(zip(self.kinds, self.steps))]
        body = [f"{a} {b}" for a, b in self.edges]
        return "\n".join(head + body) + "\n"

    @classmethod
    def from_adjacency_text(cls, text: str) -> "Dag":
        meta: dict[int, tuple[int, int]] = {}
        edges: list[tuple[int, int]] = []
        for line in (raw.strip() for raw in text.splitlines()):
            if not line:
                continue
            if line.startswith("#"):
                words = line[1:].split()
                if len(words) == 4 and words[0] == "vertex":
                    meta[int(words[1])] = (KIND_IDS[words[2]], int(words[3]))
                continue
            a, b = (int(t) for t in line.split())
            edges.append((a, b))
        n = 1 + max([*meta, *(max(e) for e in edges)], default=-1)
        dag = cls()
        for v in range(n):
            dag.add_vertex(*meta.get(v, (INTERNAL, 1)))
        for a, b in edges:
            dag.add_edge(a, b)
        return dag

    def save(self, path) -> None:
        with open(path, "w") as fh:
            fh.write(self.to_adjacency_text())

    @classmethod
    def load(cls, path) -> "Dag":
        with open(path) as fh:
            return cls.from_adjacency_text(fh.read())


@dataclass
class StepPartition:
    """Vertex sets per sub-computation step and their output subsets."""

    labels: list[int]
    step_sets: dict[int, set[int]] = field(repr=False)
    output_sets: dict[int, set[int]] = field(repr=False)

    @property
    def n_steps(self) -> int:
        return len(self.labels)


# ---------------------------------------------------------------------------
# closed-form vertex counts (the hot path's |V|)
# ---------------------------------------------------------------------------

def dc_internal_output_count(shape: ConvShape) -> int:
    """Internal + output vertices of the direct DAG: ``(2k - 1) * outputs * n``.

    Every output is one window of ``k`` products summed by a left-deep tree
    of ``k - 1`` adds.
    """
    per_output = 2 * shape.window_size - 1
    return per_output * shape.outputs_per_image * shape.n


def wa_per_tile_count(p: WinogradParams, c_in: int) -> int:
    """Vertices added by one (tile position, output channel) pair.

    Terms, in DAG step order: input-transform linear combinations, kernel
    transform linear combinations, element-wise products, channel sums,
    output transform (reference ``dag.py:190-199``).
    """
    m2 = p.m ** 2
    step1_input = m2 * (2 * m2 - 1) * c_in
    step1_kernel = m2 * (2 * p.r * p.r - 1) * c_in
    step2 = m2 * c_in
    step3 = m2 * (c_in - 1)
    step4 = p.e * p.e * (2 * m2 - 1)
    return step1_input + step1_kernel + step2 + step3 + step4


def wa_internal_output_count(shape: ConvShape, p: WinogradParams) -> int:
    pairs = (shape.w_out // p.e) * (shape.h_out // p.e) * shape.c_out
    return pairs * wa_per_tile_count(p, shape.c_in) * shape.n


def pad_shape_for_winograd(shape: ConvShape, p: WinogradParams) -> ConvShape:
    """Round the output up to a multiple of ``e``; the input grows to match."""
    def round_up(v: int) -> int:
        return ((v + p.e - 1) // p.e) * p.e

    return ConvShape.from_output(
        round_up(shape.w_out), round_up(shape.h_out), shape.c_out,
        shape.c_in, shape.w_ker, shape.h_ker, shape.stride, shape.n,
    )


# ---------------------------------------------------------------------------
# materialisation
# ---------------------------------------------------------------------------

class _Emitter:
    """Vertex-emitting helpers over one Dag (all arithmetic vertices 2-input
    sums/products or 1-input scalings)."""

    def __init__(self, dag: Dag):
        self.dag = dag

    def node(self, kind: int, step: int, *srcs: int) -> int:
        v = self.dag.add_vertex(kind, step)
        for u in srcs:
            self.dag.add_edge(u, v)
        return v

    def chain_sum(self, terms: list[int], step: int, root: int) -> int:
        """Left-deep sum; a single term is returned as is (no vertex)."""
        acc = terms[0]
        last = len(terms) - 1
        for i in range(1, len(terms)):
            acc = self.node(root if i == last else INTERNAL, step, acc, terms[i])
        return acc

    def lincomb(self, leaves: list[int], step: int, root: int) -> int:
        """Scale every leaf, then sum left-deep (2k - 2 internals + the root)."""
        lone = len(leaves) == 1
        scaled = [self.node(root if lone else INTERNAL, step, leaf) for leaf in leaves]
        return self.chain_sum(scaled, step, root)

    def input_grid(self, n: int, c: int, h: int, w: int) -> list:
        """INPUT vertices of a [n][c][h][w] tensor, nested lists."""
        return [[[[self.dag.add_vertex(INPUT, 0) for _ in range(w)] for _ in range(h)]
                 for _ in range(c)] for _ in range(n)]


def _cap_check(need: int, cap: int, what: str) -> None:
    if need > cap:
        raise SizeCapError(f"{what} needs {need} vertices, cap is {cap}")


def build_direct_conv_dag(shape: ConvShape, cap: int = DEFAULT_VERTEX_CAP) -> Dag:
    """Direct convolution (reference ``dag.py:247-285``): step 1 = every window
    product ``img[b,c,oy*mu+ky,ox*mu+kx] * wt[oc,c,ky,kx]``, step 2 = one
    left-deep sum per output over the products in ``(c, ky, kx)`` order."""
    s = shape
    n_in = s.n * s.c_in * s.h_in * s.w_in + s.c_out * s.c_in * s.h_ker * s.w_ker
    _cap_check(n_in + dc_internal_output_count(s), cap, "direct convolution dag")
    dag = Dag()
    em = _Emitter(dag)
    img = em.input_grid(s.n, s.c_in, s.h_in, s.w_in)
    wt = em.input_grid(s.c_out, s.c_in, s.h_ker, s.w_ker)
    single = s.window_size == 1
    mu = s.stride
    taps = [(c, ky, kx) for c in range(s.c_in) for ky in range(s.h_ker) for kx in range(s.w_ker)]
    for b in range(s.n):
        for oc in range(s.c_out):
            for oy in range(s.h_out):
                for ox in range(s.w_out):
                    prods = [em.node(OUTPUT if single else INTERNAL, 1,
                                     img[b][c][oy * mu + ky][ox * mu + kx], wt[oc][c][ky][kx])
                             for c, ky, kx in taps]
                    if not single:
                        em.chain_sum(prods, 2, OUTPUT)
    return dag


def build_winograd_dag(
    shape: ConvShape,
    p: WinogradParams,
    shared_kernel_transform: bool = False,
    pad: bool = False,
    cap: int = DEFAULT_VERTEX_CAP,
) -> Dag:
    """Winograd F(e x e, r x r) (reference ``dag.py:302-403``), per (image,
    output channel, tile): step 1 transforms every channel's m x m input patch
    (``img[b,c,ty*e+dy,tx*e+dx]``) and r x r kernel into m^2 values each;
    step 2 multiplies them element-wise; step 3 sums over channels; step 4
    produces the e^2 outputs.  ``shared_kernel_transform`` reuses one kernel
    transform per (output channel, channel) across tiles.
    """
    p.check_shape(shape)
    if shape.w_out % p.e or shape.h_out % p.e:
        if not pad:
            raise GeometryError(f"output {shape.w_out}x{shape.h_out} not divisible by e={p.e}; "
                                "pass pad=True to pad the output domain")
        shape = pad_shape_for_winograd(shape, p)
    s = shape
    m, m2, r2 = p.m, p.m * p.m, p.r * p.r
    ty_n, tx_n = s.h_out // p.e, s.w_out // p.e
    n_in = s.n * s.c_in * s.h_in * s.w_in + r2 * s.c_in * s.c_out
    body = wa_internal_output_count(s, p)
    if shared_kernel_transform:
        body -= (2 * r2 - 1) * m2 * s.c_in * s.c_out * s.n * (tx_n * ty_n - 1)
    _cap_check(n_in + body, cap, "winograd dag")

    dag = Dag()
    em = _Emitter(dag)
    img = em.input_grid(s.n, s.c_in, s.h_in, s.w_in)
    wt = em.input_grid(s.c_out, s.c_in, p.r, p.r)
    kernel_cache: dict[tuple[int, int], list[int]] = {}
    for b in range(s.n):
        for oc in range(s.c_out):
            for ty in range(ty_n):
                for tx in range(tx_n):
                    v_t, u_t = [], []
                    for c in range(s.c_in):
                        patch = [img[b][c][ty * p.e + dy][tx * p.e + dx]
                                 for dy in range(m) for dx in range(m)]
                        v_t.append([em.lincomb(patch, 1, INTERNAL) for _ in range(m2)])
                        if shared_kernel_transform and (oc, c) in kernel_cache:
                            u_t.append(kernel_cache[(oc, c)])
                            continue
                        kern = [wt[oc][c][ky][kx] for ky in range(p.r) for kx in range(p.r)]
                        u = [em.lincomb(kern, 1, INTERNAL) for _ in range(m2)]
                        if shared_kernel_transform:
                            kernel_cache[(oc, c)] = u
                        u_t.append(u)
                    lam = [[em.node(INTERNAL, 2, v_t[c][xi], u_t[c][xi]) for xi in range(m2)]
                           for c in range(s.c_in)]
                    pi = [em.chain_sum([lam[c][xi] for c in range(s.c_in)], 3, INTERNAL)
                          for xi in range(m2)]
                    for _ in range(p.e * p.e):
                        em.lincomb(pi, 4, OUTPUT)
    if dag.n_vertices != n_in + body:
        raise AssertionError("vertex accounting drifted")
    return dag


# ---------------------------------------------------------------------------
# multi-step partition (reference dag.py:409-457)
# ---------------------------------------------------------------------------

def validate_multi_step_partition(dag: Dag) -> StepPartition:
    """Check the multi-step partition clauses and return the partition.

    Step 0 holds exactly the primary inputs (no predecessors); every other
    vertex may read only its own step or the *outputs* of the previous
    non-empty step (primary inputs for the first one).  Empty labels are
    skipped (a one-channel Winograd DAG has no step-3 vertices).
    """
    dag.topological_order()     # cycles are a violation too
    pred = dag.predecessors()
    members: dict[int, set[int]] = {}
    for v, j in enumerate(dag.steps):
        is_input = dag.kinds[v] == INPUT
        if j == 0 and not is_input:
            raise MultiStepViolation(v, "step-0 vertex is not a primary input")
        if j == 0 and pred[v]:
            raise MultiStepViolation(v, "primary input has predecessors")
        if j != 0 and is_input:
            raise MultiStepViolation(v, "primary input carries a nonzero step label")
        if j:
            members.setdefault(j, set()).add(v)
    labels = sorted(members)
    before = dict(zip(labels, [0] + labels[:-1]))
    outs = dag.step_output_sets()
    for v, j in enumerate(dag.steps):
        if not j:
            continue
        for u in pred[v]:
            ju = dag.steps[u]
            if ju == j:
                continue
            if ju != before[j]:
                src = "a primary input" if ju == 0 else f"step {ju}"
                raise MultiStepViolation(
                    v, f"step-{j} vertex reads {src}, not an output of the previous step")
            if ju and u not in outs.get(ju, ()):
                raise MultiStepViolation(v, f"step-{j} vertex reads a non-output vertex of step {ju}")
    return StepPartition(labels, members, {j: outs.get(j, set()) for j in labels})
