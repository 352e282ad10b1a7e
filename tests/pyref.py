"""Independent pure-Python transliteration of round-synchronous SGR (pin P1).

Written from the paper's pseudocode without looking at oracle.c's control flow:
sets and dicts instead of stamped arrays and worklist buffers.  Used only on tiny
graphs (exhaustive <= 6 vertices) to cross-check the C oracle.

  Alg. 2 / Alg. 7, FirstFit,
  ConflictResolve, §3.2 degree heuristic.
"""
from itertools import count


def loser_of(v, w, policy, deg):
    """Which endpoint of a same-colour edge {v, w} recolours."""
    if policy == "higher_id":
        return max(v, w)
    if policy == "lower_id":
        return min(v, w)
    # degree: smaller degree recolours; tie -> the smaller id is "picked" (keeps colour)
    if deg[v] != deg[w]:
        return v if deg[v] < deg[w] else w
    return max(v, w)


def sgr(n, adj, policy="higher_id"):
    """adj: list of sets.  Returns (colors list, num_colors, rounds, trace)."""
    deg = [len(a) for a in adj]
    final = {}
    pending = set(range(n))
    rounds = 0
    trace = []
    while pending:
        rounds += 1
        trace.append(len(pending))
        tent = {}
        for v in pending:
            forbidden = {final[w] for w in adj[v] if w in final}
            tent[v] = next(c for c in count(1) if c not in forbidden)
        losers = set()
        for v in pending:
            for w in adj[v]:
                if w in pending and tent[w] == tent[v]:
                    losers.add(loser_of(v, w, policy, deg))
        for v in pending - losers:
            final[v] = tent[v]
        pending = losers
    colors = [final[v] for v in range(n)]
    return colors, (max(colors) if colors else 0), rounds, trace


def greedy(n, adj):
    """Alg. 1 in ascending id order."""
    col = [0] * n
    for v in range(n):
        used = {col[w] for w in adj[v]}
        col[v] = next(c for c in count(1) if c not in used)
    return col


def adj_of(g):
    return [set(int(x) for x in g.col_idx[g.row_ptr[v]:g.row_ptr[v + 1]]) for v in range(g.n)]
