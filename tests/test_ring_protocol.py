"""Happens-before check of the push-form ring reduce-scatter's buffer protocol
(paper_2008_00177_b200/csrc/bo_ring.cu ring_reduce_scatter, push branch) for
every world size the library supports, 2..8 — including the 8-GPU world that
the development GPU pool cannot grant.

Model. Rank r runs, in stream order: hop 0 (pack: write the right
neighbour's staging buffer 0), then for s = 0..N-2: barrier B_s, hop s+1
(read own buffer s % 2; write the right neighbour's buffer (s+1) % 2, or its
own buffer (N-1) % 2 on the last hop — or, with the last hop fused into LAMB
phase 1, read own buffer (N-2) % 2 there). B_s is the neighbour barrier
(k_ring_barrier): rank r leaves B_s only after both ring neighbours have
arrived at it, i.e. finished everything before their own B_s. An access of
rank x in segment i (between B_{i-1} and B_i; segment 0 is before B_0) is
therefore ordered before an access of rank y in segment k when k >= i + d,
d >= 1 the ring distance from x to y (one neighbour hop per barrier), or
when x == y and the access comes later in program order. Every pair of
conflicting accesses (same buffer, at least one write) within a step must be
ordered. Across steps, `test_consecutive_steps_*` adds the step's all-rank
flag barriers (the partials barrier in k_trust after LAMB phase 1, the
end-of-step barrier after the parameter push): nothing else separates step t's
last read of a staging buffer from step t+1's hop-0 push into it.
"""
import itertools

import pytest


def accesses(N, fuse_last):
    """[(rank, segment, order, owner, buffer, kind)] of one step."""
    acc = []
    for r in range(N):
        right = (r + 1) % N
        order = 0
        acc.append((r, 0, order, right, 0, "w"))  # hop 0: push chunk r
        for s in range(N - 1):
            seg = s + 1  # after B_s
            order += 1
            acc.append((r, seg, order, r, s % 2, "r"))
            if s == N - 2 and fuse_last:
                continue  # LAMB phase 1 reads the input in place, writes nothing here
            if s == N - 2:
                acc.append((r, seg, order, r, (s + 1) % 2, "w"))  # last hop: the owned chunk, locally
            else:
                acc.append((r, seg, order, right, (s + 1) % 2, "w"))
        # LAMB phase 1 (unfused) reads the final buffer after the last hop
        if not fuse_last:
            acc.append((r, N - 1, order + 1, r, (N - 1) % 2, "r"))
    return acc


def ring_dist(x, y, N):
    return min((y - x) % N, (x - y) % N)


def ordered(a, b, N):
    """True when access a happens before access b under the neighbour barriers."""
    xa, ia, oa = a[0], a[1], a[2]
    xb, ib, ob = b[0], b[1], b[2]
    if xa == xb:
        return (ib, ob) > (ia, oa)
    return ib >= ia + ring_dist(xa, xb, N)


@pytest.mark.parametrize("N", range(2, 9))
@pytest.mark.parametrize("fuse_last", [False, True])
def test_push_ring_buffers_race_free(N, fuse_last):
    acc = accesses(N, fuse_last)
    for a, b in itertools.combinations(acc, 2):
        if (a[3], a[4]) != (b[3], b[4]) or (a[5] == "r" and b[5] == "r"):
            continue
        if a[0] == b[0] and a[1] == b[1] and a[2] == b[2]:
            continue  # one hop kernel reading and writing different elements of one buffer: not a pair here
        assert ordered(a, b, N) or ordered(b, a, N), (N, fuse_last, a, b)


@pytest.mark.parametrize("N", range(2, 9))
def test_every_read_sees_the_pushed_partial(N):
    """Rank r's hop s+1 reads buffer s % 2 of its own memory, which the left
    neighbour's hop s (or pack) wrote in the previous segment — the chunk
    fold order of collective.hpp:65-80 (chunk k folds ranks k, k+1, ...)."""
    acc = accesses(N, False)
    for r in range(N):
        left = (r - 1) % N
        for s in range(N - 1):
            read = next(a for a in acc if a[0] == r and a[1] == s + 1 and a[5] == "r")
            writes = [a for a in acc if a[3] == r and a[4] == s % 2 and a[5] == "w" and a[0] == left]
            last = max((w for w in writes if ordered(w, read, N)), key=lambda w: (w[1], w[2]))
            assert last[1] == s  # the left neighbour's previous hop


@pytest.mark.parametrize("N", [4, 8])
def test_waiting_for_the_left_neighbour_alone_would_race(N):
    """Why k_ring_barrier waits for BOTH neighbours: with the left one alone, a
    rank could push into its right neighbour's buffer while that neighbour
    still reads the previous partial from it (write-after-read)."""

    def ordered_left_only(a, b):
        if a[0] == b[0]:
            return (b[1], b[2]) > (a[1], a[2])
        return b[1] >= a[1] + (b[0] - a[0]) % N

    acc = accesses(N, False)
    races = [(a, b) for a, b in itertools.combinations(acc, 2)
             if (a[3], a[4]) == (b[3], b[4]) and "w" in (a[5], b[5])
             and not (a[0] == b[0] and a[1] == b[1] and a[2] == b[2])
             and not (ordered_left_only(a, b) or ordered_left_only(b, a))]
    assert races and all({a[5], b[5]} == {"r", "w"} for a, b in races)


def accesses_pull(N, fuse_last):
    """The pull form (BO_RING_PUSH=0): hop 0 packs into the own buffer 0; hop s
    reads the LEFT neighbour's buffer s % 2 in place and writes its own
    buffer (s+1) % 2; a fused last hop reads the left's buffer inside phase 1."""
    acc = []
    for r in range(N):
        left = (r - 1) % N
        order = 0
        acc.append((r, 0, order, r, 0, "w"))
        for s in range(N - 1):
            seg = s + 1
            order += 1
            acc.append((r, seg, order, left, s % 2, "r"))
            if s == N - 2 and fuse_last:
                continue
            acc.append((r, seg, order, r, (s + 1) % 2, "w"))
        if not fuse_last:
            acc.append((r, N - 1, order + 1, r, (N - 1) % 2, "r"))
    return acc


@pytest.mark.parametrize("N", range(2, 9))
@pytest.mark.parametrize("fuse_last", [False, True])
def test_pull_ring_buffers_race_free(N, fuse_last):
    acc = accesses_pull(N, fuse_last)
    for a, b in itertools.combinations(acc, 2):
        if (a[3], a[4]) != (b[3], b[4]) or (a[5] == "r" and b[5] == "r"):
            continue
        if a[0] == b[0] and a[1] == b[1] and a[2] == b[2]:
            continue
        assert ordered(a, b, N) or ordered(b, a, N), (N, fuse_last, a, b)


def accesses_steps(N, fuse_last, steps, groups):
    """Several consecutive steps, the reduce-scatter of each step split into
    `groups` communication groups (the overlapped sync micro: every group's
    hops run on the communication stream, group after group, each with its own
    neighbour barriers; groups own disjoint buckets, i.e. disjoint slices of
    the staging buffers). Returns (accesses, barrier kinds): an access is
    (rank, segment, order, owner, (group, buffer), kind); kinds[j] is "nb"
    (neighbour) or "all" (all-rank) for the barrier ending segment j."""
    acc, kinds = [], []
    seg = 0
    order = 0
    for _t in range(steps):
        for g in range(groups):
            fuse = fuse_last and groups == 1  # the overlapped sync micro stages its last hop
            for r in range(N):
                acc.append((r, seg, order, (r + 1) % N, (g, 0), "w"))  # hop 0
            for s in range(N - 1):
                kinds.append("nb")
                seg += 1
                order += 1
                for r in range(N):
                    right = (r + 1) % N
                    acc.append((r, seg, order, r, (g, s % 2), "r"))
                    if s == N - 2 and fuse:
                        continue
                    owner = r if s == N - 2 else right
                    acc.append((r, seg, order, owner, (g, (s + 1) % 2), "w"))
            order += 1
            # LAMB phase 1 reads the reduced chunk (fused: the last hop's input)
            for r in range(N):
                acc.append((r, seg, order, r, (g, (N - 2) % 2 if fuse else (N - 1) % 2), "r"))
        kinds.append("all")  # k_trust: partials barrier (after every rank's phase 1)
        seg += 1
        kinds.append("all")  # end-of-step barrier (after every rank's parameter push)
        seg += 1
        order += 1
    return acc, kinds


def ordered_steps(a, b, N, kinds):
    xa, ia, oa = a[0], a[1], a[2]
    xb, ib, ob = b[0], b[1], b[2]
    if xa == xb:
        return (ib, ob) > (ia, oa)
    if ib <= ia:
        return False
    if any(k == "all" for k in kinds[ia:ib]):
        return True
    return ib >= ia + ring_dist(xa, xb, N)


@pytest.mark.parametrize("N", range(2, 9))
@pytest.mark.parametrize("fuse_last", [False, True])
@pytest.mark.parametrize("groups", [1, 3])
def test_consecutive_steps_race_free(N, fuse_last, groups):
    """Two consecutive steps (and overlapped communication groups): the next
    step's hop-0 push into the right neighbour's staging buffer 0 is ordered
    after that neighbour's last read of it in the previous step only through
    the previous step's partials barrier (bo_ring.cu, hop 0 comment)."""
    acc, kinds = accesses_steps(N, fuse_last, 2, groups)
    for a, b in itertools.combinations(acc, 2):
        if (a[3], a[4]) != (b[3], b[4]) or (a[5] == "r" and b[5] == "r"):
            continue
        if a[0] == b[0] and a[1] == b[1] and a[2] == b[2]:
            continue
        assert ordered_steps(a, b, N, kinds) or ordered_steps(b, a, N, kinds), (N, fuse_last, a, b)


@pytest.mark.parametrize("N", [2, 4, 6, 8])
def test_consecutive_steps_need_the_partials_barrier(N):
    """Negative control: drop the step's all-rank barriers and, at every even
    world, the next step's hop 0 pushes into staging buffer 0 while the right
    neighbour's fused last hop ((N-2) % 2 == 0) may still read it in phase 1
    (the dependency the hop-0 comment in bo_ring.cu documents)."""
    acc, kinds = accesses_steps(N, True, 2, 1)
    cut = [i for i, k in enumerate(kinds) if k == "all"]
    acc = [(x, seg - sum(1 for j in cut if j < seg), o, ow, buf, kd) for (x, seg, o, ow, buf, kd) in acc]
    kinds = [k for k in kinds if k != "all"]
    races = [(a, b) for a, b in itertools.combinations(acc, 2)
             if (a[3], a[4]) == (b[3], b[4]) and "w" in (a[5], b[5])
             and not (a[0] == b[0] and a[1] == b[1] and a[2] == b[2])
             and not (ordered_steps(a, b, N, kinds) or ordered_steps(b, a, N, kinds))]
    assert races and all(b[4] == (0, 0) and {a[5], b[5]} == {"r", "w"} for a, b in races)
