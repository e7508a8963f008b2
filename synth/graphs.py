"""Seeded heterograph generators and the G7 fixture.

Graph conventions:
  * global node ids; node type t owns the contiguous id range
    [node_type_ptr[t], node_type_ptr[t+1])  ("nodes are presorted", §3.4.1;
    S:115 graph-core External Interfaces);
  * an edge e is (src[e], dst[e], rel[e]); edge ids are positions in these arrays.

Generator recipe: node-type sizes Zipf(1.0) over types
(>=1 node each) when only T is known; each relation draws a canonical
(src_type, dst_type) proportionally to type sizes; relation sizes
E_r ~ Multinomial(E, Zipf(1.0)); within relation r sources follow Zipf(a_src)
over a seeded permutation of the source-type nodes and destinations follow
Zipf(a_dst) over a seeded permutation of the destination-type nodes;
duplicate (src, dst, rel) triples are redrawn.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


@dataclasses.dataclass
class HeteroGraph:
    node_type_ptr: np.ndarray          # int64 [T+1]
    num_rels: int
    src: np.ndarray                    # int32 [E]
    dst: np.ndarray                    # int32 [E]
    rel: np.ndarray                    # int32 [E]
    name: str = ""
    rel_types: Optional[np.ndarray] = None   # int32 [R, 2] canonical (src_type, dst_type), informative

    @property
    def num_nodes(self) -> int:
        return int(self.node_type_ptr[-1])

    @property
    def num_node_types(self) -> int:
        return int(len(self.node_type_ptr) - 1)

    @property
    def num_edges(self) -> int:
        return int(len(self.src))

    def node_type_of(self) -> np.ndarray:
        """Node type per node id (int32 [N])."""
        counts = np.diff(self.node_type_ptr)
        return np.repeat(np.arange(self.num_node_types, dtype=np.int32), counts)

    def validate(self) -> None:
        n = self.num_nodes
        if self.num_edges:
            if self.src.min() < 0 or self.src.max() >= n or self.dst.min() < 0 or self.dst.max() >= n:
                raise ValueError("node id out of range")
            if self.rel.min() < 0 or self.rel.max() >= self.num_rels:
                raise ValueError("relation id out of range")


# ---------------------------------------------------------------- G7 fixture
G7_TSV = """# G7 fixture, SPEC.md S:115 (graph-core External Interfaces)
# authors a=0,b=1,c=2 ; papers p=3,q=4 ; writes=0, cites=1
H 2 2
N 3 2
E 0 3 0
E 0 4 0
E 1 3 0
E 1 4 0
E 2 4 0
E 3 4 1
E 4 3 1
"""


def load_tsv(text: str, name: str = "") -> HeteroGraph:
    """Parse the S:115 graph-TSV format.  Errors carry the 1-based line number."""
    header = None
    counts = None
    src: List[int] = []
    dst: List[int] = []
    rel: List[int] = []
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        try:
            if tok[0] == "H":
                if header is not None:
                    raise ValueError(f"duplicate header at line {ln}")
                header = (int(tok[1]), int(tok[2]))
            elif tok[0] == "N":
                counts = [int(t) for t in tok[1:]]
                if header is None or len(counts) != header[0]:
                    raise ValueError(f"malformed N line at line {ln}")
            elif tok[0] == "E":
                if counts is None or len(tok) != 4:
                    raise ValueError(f"malformed E line at line {ln}")
                s, d, r = int(tok[1]), int(tok[2]), int(tok[3])
                n = sum(counts)
                if not (0 <= s < n and 0 <= d < n and 0 <= r < header[1]):
                    raise ValueError(f"id out of range at line {ln}")
                src.append(s); dst.append(d); rel.append(r)
            else:
                raise ValueError(f"malformed line at line {ln}")
        except (IndexError, ValueError) as exc:
            if "line" in str(exc):
                raise
            raise ValueError(f"malformed line at line {ln}") from exc
    if header is None or counts is None:
        raise ValueError("missing H or N line")
    ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    g = HeteroGraph(ptr, header[1], np.asarray(src, np.int32), np.asarray(dst, np.int32),
                    np.asarray(rel, np.int32), name=name)
    return g


def dump_tsv(g: HeteroGraph) -> str:
    lines = [f"H {g.num_node_types} {g.num_rels}",
             "N " + " ".join(str(int(c)) for c in np.diff(g.node_type_ptr))]
    lines += [f"E {int(s)} {int(d)} {int(r)}" for s, d, r in zip(g.src, g.dst, g.rel)]
    return "\n".join(lines) + "\n"


def g7() -> HeteroGraph:
    return load_tsv(G7_TSV, name="G7")


# ---------------------------------------------------------------- sampling helpers
def _zipf_probs(n: int, a: float) -> np.ndarray:
    k = np.arange(1, n + 1, dtype=np.float64)
    w = k ** (-a) if a != 0.0 else np.ones(n)
    return w / w.sum()


def _zipf_sampler(n: int, a: float):
    cdf = np.cumsum(_zipf_probs(n, a))
    cdf[-1] = 1.0

    def draw(rng: np.random.Generator, size: int) -> np.ndarray:
        u = rng.random(size)
        return np.minimum(np.searchsorted(cdf, u, side="right"), n - 1)
    return draw


def _type_sizes(n: int, t: int) -> np.ndarray:
    p = _zipf_probs(t, 1.0)
    sizes = np.maximum(1, np.floor(n * p).astype(np.int64))
    sizes[0] += n - sizes.sum()
    if sizes[0] < 1:
        raise ValueError("infeasible node-type split")
    return sizes


def _relation_sizes(rng, e: int, caps: np.ndarray) -> np.ndarray:
    """E_r ~ Multinomial(E, Zipf(1.0)) clipped to the per-relation capacity
    (distinct (src,dst) pairs), excess redistributed the same way."""
    r = len(caps)
    if caps.sum() < e:
        raise ValueError(f"infeasible spec: {e} distinct edges requested, at most {caps.sum()} possible")
    p = _zipf_probs(r, 1.0)
    sizes = rng.multinomial(e, p).astype(np.int64)
    for _ in range(1000):
        over = np.maximum(0, sizes - caps)
        excess = int(over.sum())
        sizes -= over
        if excess == 0:
            return sizes
        room = caps - sizes
        q = p * (room > 0)
        q = q / q.sum()
        add = rng.multinomial(excess, q)
        sizes += add
    raise ValueError("could not place relation sizes")


def synth_heterograph(type_sizes: Sequence[int], rel_types: Sequence[Tuple[int, int]],
                      rel_sizes: Optional[Sequence[int]] = None, num_edges: Optional[int] = None,
                      a_src: float = 0.5, a_dst: float = 0.8, seed: int = 1,
                      name: str = "synthetic", max_rounds: int = 400) -> HeteroGraph:
    """Draw a heterograph.  Deterministic per seed; raises
    ValueError on an infeasible spec."""
    rng = np.random.default_rng(seed)
    type_sizes = np.asarray(type_sizes, np.int64)
    ptr = np.concatenate([[0], np.cumsum(type_sizes)]).astype(np.int64)
    n = int(ptr[-1])
    rel_types = np.asarray(rel_types, np.int32).reshape(-1, 2)
    r = len(rel_types)
    caps = type_sizes[rel_types[:, 0]] * type_sizes[rel_types[:, 1]]
    if rel_sizes is None:
        rel_sizes = _relation_sizes(rng, int(num_edges), caps)
    rel_sizes = np.asarray(rel_sizes, np.int64)
    if np.any(rel_sizes > caps):
        raise ValueError("infeasible spec: relation larger than its distinct (src,dst) capacity")
    # one seeded permutation per node type: Zipf rank -> node (hubs land on random ids)
    perms = [rng.permutation(int(s)).astype(np.int64) for s in type_sizes]
    samplers: Dict[Tuple[int, float], object] = {}

    def sampler(t: int, a: float):
        key = (t, a)
        if key not in samplers:
            samplers[key] = _zipf_sampler(int(type_sizes[t]), a)
        return samplers[key]

    srcs, dsts, rels = [], [], []
    for ri in range(r):
        er = int(rel_sizes[ri])
        if er == 0:
            continue
        st, dt = int(rel_types[ri, 0]), int(rel_types[ri, 1])
        ds, dd = sampler(st, a_src), sampler(dt, a_dst)
        nd = int(type_sizes[dt])
        keys = np.empty(0, np.int64)
        for _ in range(max_rounds):
            need = er - len(keys)
            if need == 0:
                break
            # oversample a little to converge in few rounds on skewed relations
            m = need + need // 8 + 16
            s = perms[st][ds(rng, m)]
            d = perms[dt][dd(rng, m)]
            new = s * nd + d
            # keep first occurrences in draw order (deterministic)
            allk = np.concatenate([keys, new])
            _, first = np.unique(allk, return_index=True)
            first.sort()
            keys = allk[first][:er]
        else:
            raise ValueError(f"relation {ri}: could not draw {er} distinct edges")
        srcs.append((keys // nd + ptr[st]).astype(np.int32))
        dsts.append((keys % nd + ptr[dt]).astype(np.int32))
        rels.append(np.full(er, ri, np.int32))
    if srcs:
        src = np.concatenate(srcs); dst = np.concatenate(dsts); rel = np.concatenate(rels)
        # interleave relations: a seeded shuffle of the edge order (edge ids are arbitrary)
        order = rng.permutation(len(src))
        src, dst, rel = src[order], dst[order], rel[order]
    else:
        src = dst = rel = np.zeros(0, np.int32)
    g = HeteroGraph(ptr, r, src, dst, rel, name=name, rel_types=rel_types)
    g.validate()
    return g


def _draw_rel_types(rng, type_sizes: np.ndarray, r: int) -> np.ndarray:
    p = type_sizes / type_sizes.sum()
    return np.stack([rng.choice(len(type_sizes), size=r, p=p),
                     rng.choice(len(type_sizes), size=r, p=p)], axis=1).astype(np.int32)


# ---------------------------------------------------------------- configs
# Shapes: tab:datasets P:1032-1043; AM follows BASELINE.json (reading g14);
# mag type/relation sizes follow public ogbn-mag statistics (outside the paper,
# SURVEY.md §8(d) D1 table, unpinned).
CONFIGS: Dict[str, dict] = {
    "tiny":    dict(nodes=1000, types=4, rels=8, edges=10_000, a_src=0.5, a_dst=0.8, equal_types=True),
    "aifb":    dict(nodes=7_300, types=7, rels=104, edges=49_000, a_src=0.5, a_dst=0.8),
    "mutag":   dict(nodes=27_000, types=5, rels=50, edges=148_000, a_src=0.5, a_dst=0.8),
    "bgs":     dict(nodes=95_000, types=27, rels=122, edges=673_000, a_src=0.5, a_dst=0.8),
    "am":      dict(nodes=900_000, types=7, rels=130, edges=5_700_000, a_src=0.3, a_dst=0.8),
    "fb15k":   dict(nodes=15_000, types=1, rels=474, edges=620_000, a_src=1.15, a_dst=0.8),
    "biokg":   dict(nodes=94_000, types=5, rels=51, edges=4_800_000, a_src=0.5, a_dst=0.8),
    "wikikg2": dict(nodes=2_500_000, types=1, rels=535, edges=16_000_000, a_src=0.5, a_dst=0.8),
    "mag":     dict(type_sizes=[736_389, 1_134_649, 8_740, 59_965],
                    # (src_type, dst_type): writes author->paper, cites paper->paper,
                    # has_topic paper->field, affiliated_with author->institution
                    rel_types=[(1, 0), (0, 0), (0, 3), (1, 2)],
                    rel_sizes=[7_145_660, 5_416_271, 7_505_078, 1_043_998],
                    a_src=0.5, a_dst=0.8),
}


def config_graph(name: str, seed: int = 1, scale: float = 1.0, a_dst: Optional[float] = None) -> HeteroGraph:
    """Graph for a named config.  `scale` (<1) shrinks nodes and edges
    proportionally (used for oracle-sized parity cases)."""
    spec = dict(CONFIGS[name])
    if a_dst is not None:
        spec["a_dst"] = a_dst
    rng = np.random.default_rng(seed + 1_000_003)
    if "type_sizes" in spec:
        ts = np.maximum(1, np.round(np.asarray(spec["type_sizes"]) * scale)).astype(np.int64)
        rs = np.maximum(1, np.round(np.asarray(spec["rel_sizes"]) * scale)).astype(np.int64)
        return synth_heterograph(ts, spec["rel_types"], rel_sizes=rs, a_src=spec["a_src"],
                                 a_dst=spec["a_dst"], seed=seed, name=name if scale == 1.0 else f"{name}@{scale:g}")
    n = max(spec["types"], int(round(spec["nodes"] * scale)))
    e = max(1, int(round(spec["edges"] * scale)))
    if spec.get("equal_types"):
        ts = np.full(spec["types"], n // spec["types"], np.int64)
        ts[0] += n - ts.sum()
    else:
        ts = _type_sizes(n, spec["types"])
    rt = _draw_rel_types(rng, ts, spec["rels"])
    return synth_heterograph(ts, rt, num_edges=e, a_src=spec["a_src"], a_dst=spec["a_dst"],
                             seed=seed, name=name if scale == 1.0 else f"{name}@{scale:g}")


def random_small_graph(seed: int, max_nodes: int = 32, max_edges: int = 128, max_rels: int = 4,
                       max_types: int = 3, allow_multi: bool = False) -> HeteroGraph:
    """Random-graph suite member (S:606 limits: <=32 nodes, <=128 edges, <=4 etypes).
    Uniform endpoints; includes isolated nodes and empty relations by chance."""
    rng = np.random.default_rng(seed)
    t = int(rng.integers(1, max_types + 1))
    n = int(rng.integers(max(t, 2), max_nodes + 1))
    cuts = np.sort(rng.choice(np.arange(1, n), size=t - 1, replace=False)) if t > 1 else np.zeros(0, np.int64)
    ptr = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    r = int(rng.integers(1, max_rels + 1))
    e = int(rng.integers(0, max_edges + 1))
    src = rng.integers(0, n, size=e).astype(np.int32)
    dst = rng.integers(0, n, size=e).astype(np.int32)
    rel = rng.integers(0, r, size=e).astype(np.int32)
    if not allow_multi and e:
        key = (src.astype(np.int64) * n + dst) * r + rel
        _, first = np.unique(key, return_index=True)
        first.sort()
        src, dst, rel = src[first], dst[first], rel[first]
    return HeteroGraph(ptr, r, src, dst, rel, name=f"rand{seed}")
