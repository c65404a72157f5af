"""Hand-traced pins for the parts of the oracle planner / simulator whose earlier tests were
order-insensitive (VERDICT r01 "weak" 1): the step-1 scan order ("in order from the
output layer"), the L_I tree cap and its overflow (Reading 16), the Fig. 13 search size
(P:L274), the NAIVE swap-in trigger (Reading 8), the SuperNeurons trigger
 and the host-capacity start of step 1 (Reading 37).

Every expected value below was derived by hand from the rules quoted in oracle/sim.py and
oracle/planner.py on the Fig. 11 chain of tests/golden/fig11_chain.json (8 tasks, fwd 10,
bwd 10 except bwd(7) = 20, every map 1 byte, d2h 5 except map 5 = 15, h2d 5 except map 4 = 40,
task i reads map i-1, bwd(i) needs {i-1, i}); the derivations are written next to them.

All-swap, eager, unlimited memory (the base timeline every step-1 case starts from):
  F_i = [10i, 10i+10], forward ends at 80. Swap-out of m is ready when F_{m+1} ends (m < 7),
  of the sink when F_7 ends: O0 [20,25] O1 [30,35] O2 [40,45] O3 [50,55] O4 [60,65]
  O5 [70,85] O6 [85,90] O7 [90,95] (O6, O7 both ready at 80: smaller id first).
  Need order (first backward user): maps 6, 7 -> B7 (program pos 8); 5 -> B6; 4 -> B5; ...
  Swap-ins FIFO 6, 7, 5, 4, 3, 2, 1, 0 once forward has ended and the swap-out is done:
  I6 [90,95] I7 [95,100] I5 [100,105] I4 [105,145] I3 [145,150] I2 [150,155] I1 [155,160]
  I0 [160,165]. Backward: B7 [100,120] B6 [120,130] B5 [145,155] B4 [155,165] B3 [165,175]
  B2 [175,185] B1 [185,195] B0 [195,205]: makespan 205.
  Stall = swap-in end - end of the program task before the first user:
  map 7: 100 - 80 = 20; map 6: 95 - 80 = 15; map 4: 145 - 130 = 15; map 5: 105 - 120 < 0 -> 0;
  maps 3..0: 0. So L_O = {5, 6, 7} (swap-outs ending after 80), L_I = {4, 6, 7} -- the
  paper's sets -- and the stall ranking is 7 (20), 4 (15), 6 (15; tie -> smaller id).
"""
import json
import os

import pytest

from oracle import planner
from oracle.sim import EAGER, KEEP, NAIVE, RECOMPUTE, SN, SWAP, Profile, simulate

G = os.path.join(os.path.dirname(__file__), "golden")


def _fig11(**kw):
    return Profile.from_dict(json.load(open(os.path.join(G, "fig11_chain.json"))), **kw)


def _cls(keeps):
    c = [SWAP] * 8
    for m in keeps:
        c[m] = KEEP
    return tuple(c)


def test_fig11_stalls_by_hand():
    r = simulate(_fig11(), [SWAP] * 8)
    assert r.makespan == 205
    assert r.stall == {7: 20, 6: 15, 4: 15, 5: 0, 3: 0, 2: 0, 1: 0, 0: 0}


@pytest.mark.parametrize("li_cap, tree, scan, sims", [
    # cap >= |L_I| = 3: tree L_I = {4,6,7}, scan L_O \ L_I = {5}: Fig. 13's 2^3 leaves, each
    # simulated once and followed by the one-element scan -> 1 + 8 * (1 + 1) = 17 simulations
    (3, [4, 6, 7], [5], 17),
    (16, [4, 6, 7], [5], 17),
    # cap 2: the two largest stalls (7: 20; 4 beats 6 on the tie by id) form the tree; the
    # overflow {6} joins the scan, which runs from the output layer: [6, 5] -> 1 + 4 * 3 = 13
    (2, [4, 7], [6, 5], 13),
    # cap 1: tree {7}; scan {5,6} u overflow {4,6} from the output side: [6, 5, 4] -> 1 + 2 * 4 = 9
    (1, [7], [6, 5, 4], 9),
    # cap 0: no tree, one leaf; scan L_O u L_I from the output side: [7, 6, 5, 4] -> 1 + 5 = 6
    (0, [], [7, 6, 5, 4], 6),
])
def test_step1_tree_scan_and_search_size(li_cap, tree, scan, sims):
    log = []
    cls, ms, n = planner.step1(_fig11(), li_cap, log=log)
    tag, lo, li, t, s, best = log[0]
    assert (lo, li) == ([5, 6, 7], [4, 6, 7])
    assert t == tree and s == scan
    assert n == sims


def test_step1_visits_from_the_output_layer():
    """cap 0, unlimited memory: after the start and the (only, empty-tree) leaf, the scan keeps 7,
    then 6, 5, 4. Each
    state's makespan, by hand (swap-ins start at 80 unless their swap-out ends later):
      keep {7}:        I6 [90,95] I5 [95,100] I4 [100,140] I3..I0 five-apart to 160;
                       B7 [95,115] B6 [115,125] B5 [140,150] B4 [150,160] ... B0 [190,200] -> 200
      keep {7,6}:      I5 [85,90] I4 [90,130] ...; B7 [80,100] B6 [100,110] B5 [130,140] ... -> 190
      keep {7,6,5}:    I4 [80,120] ...; B7 [80,100] B6 [100,110] B5 [120,130] ... B0 [170,180] -> 180
      keep {7,6,5,4}:  I3 [80,85] .. I0 [95,100]; B7 [80,100] B6 .. B4 [120,130] .. B0 [160,170] -> 170
    An input-first scan would visit keep {4} second."""
    trace = []
    cls, ms, _ = planner.step1(_fig11(), 0, trace=trace)
    assert trace == [(_cls([]), 205), (_cls([]), 205), (_cls([7]), 200), (_cls([7, 6]), 190), (_cls([7, 6, 5]), 180),
                     (_cls([7, 6, 5, 4]), 170)]
    assert tuple(cls) == _cls([7, 6, 5, 4]) and ms == 170


def test_step1_cap2_leaf_order_and_choice():
    """cap 2: tree [4, 7] (bit b of the leaf number keeps tree[b]); each leaf scans 6 then 5.
    The chosen state keeps {4, 6, 7} and swaps 5: O5 [70,85], I5 [85,90], I3 [90,95] .. I0
    [105,110]; B7 [80,100] B6 [100,110] B5 [110,120] B4 [120,130] .. B0 [160,170] -> 170, the
    same makespan as keeping all four, with one keep fewer (tie-break on #keep, Reading 19)."""
    trace = []
    cls, ms, _ = planner.step1(_fig11(), 2, trace=trace)
    visited = [tuple(m for m in range(8) if c[m] == KEEP) for c, _ in trace]
    assert visited == [(),
                       (), (6,), (5, 6),                    # leaf 0
                       (4,), (4, 6), (4, 5, 6),             # leaf 1: keep tree[0] = 4
                       (7,), (6, 7), (5, 6, 7),             # leaf 2: keep tree[1] = 7
                       (4, 7), (4, 6, 7), (4, 5, 6, 7)]     # leaf 3
    assert tuple(cls) == _cls([4, 6, 7]) and ms == 170


def _swapins(r):
    return [(i, s, e) for lane, k, i, s, e in r.events if k == "I"]


def test_naive_swapin_by_hand():
    """NAIVE (P:L109 / P:L353; Reading 8): swap-in of m may start when the program task just
    before m's first backward user starts (and its swap-out is done, the H2D lane free).
      6, 7 (first user B7, preceded by F7, started at 70): I6 at O6's end 90, I7 at 95;
      5 (user B6, preceded by B7 which starts at 100): I5 [100,105];
      4 (user B5; B6 starts at 120 once B7 ends): I4 [120,160];
      3 (user B4; B5 waits for I4 -> starts 160): I3 [160,165];
      2 (B3; B4 starts at B5's end 170): I2 [170,175];  1 (B2; B3 at 180): I1 [180,185];
      0 (B1; B2 at 190): I0 [190,195];  B1 [200,210], B0 [210,220] -> makespan 220."""
    r = simulate(_fig11(), [SWAP] * 8, NAIVE)
    assert _swapins(r) == [(6, 90, 95), (7, 95, 100), (5, 100, 105), (4, 120, 160), (3, 160, 165),
                           (2, 170, 175), (1, 180, 185), (0, 190, 195)]
    assert r.makespan == 220


def test_superneurons_swapin_by_hand():
    """SuperNeurons ("each swap-in starts simultaneously with the computation of the
    immediately preceding convolution layer"), with tasks 0, 2, 4, 6 convolutions: the trigger of
    m is the latest convolution backward before m's first user (the last forward task when there
    is none).  6, 7, 5: F7 (70) -> I6 [90,95], I7 [95,100], I5 [100,105];  4 (user B5): B6 (conv)
    starts 120 -> I4 [120,160];  3 (user B4): B6 again -> right after I4, [160,165];  2 (user B3):
    B4 (conv) starts 170 -> [170,175];  1 (user B2): B4 again -> [175,180] (five earlier than
    NAIVE);  0 (user B1): B2 (conv) starts 190 -> [190,195] -> makespan 220."""
    d = json.load(open(os.path.join(G, "fig11_chain.json")))
    d["is_conv"] = [1, 0, 1, 0, 1, 0, 1, 0]
    r = simulate(Profile.from_dict(d), [SWAP] * 8, SN)
    assert _swapins(r) == [(6, 90, 95), (7, 95, 100), (5, 100, 105), (4, 120, 160), (3, 160, 165),
                           (2, 170, 175), (1, 175, 180), (0, 190, 195)]
    assert r.makespan == 220


def test_eager_swapin_by_hand():
    """EAGER: every swap-in as early as the lane, its swap-out and the memory gate allow
    once forward is over (module docstring trace)."""
    r = simulate(_fig11(), [SWAP] * 8, EAGER)
    assert _swapins(r) == [(6, 90, 95), (7, 95, 100), (5, 100, 105), (4, 105, 145), (3, 145, 150),
                           (2, 150, 155), (1, 155, 160), (0, 160, 165)]


def test_host_fit_base_by_hand():
    """Reading 37: when all-swap's swap class exceeds the host arena, step 1 starts from all-swap
    with the maps of cheapest replay per byte moved to recompute (ties: larger bytes first, then
    smaller id; never the sink) until the swap class fits.
      bytes [4, 2, 8, 4], rec [8, 1, 4, 1] -> rec/byte 2, 0.5, 0.5, (sink 0.25: never moved);
      total 18. Host 10: order m2 (0.5, 8 B) before m1 (0.5, 2 B) -> moving m2 leaves 10 <= 10:
      [swap, swap, recompute, swap]. Host 9: m2 then m1 -> 8: [swap, recompute, recompute, swap].
      Host 3: m2, m1, m0 -> 4 > 3 with only the sink left, which cannot be recompute:
      it is kept -> [rec, rec, rec, keep]; likewise with no host arena at all (0 bytes)."""
    def prof(host):
        return Profile([1] * 4, [1] * 4, [4, 2, 8, 4], [1] * 4, [1] * 4, [[], [0], [1], [2]],
                       [[0], [1], [2], [3]], rec=[8, 1, 4, 1], host_budget=host)
    assert planner.host_fit_base(prof(None)) == [SWAP] * 4
    assert planner.host_fit_base(prof(18)) == [SWAP] * 4
    assert planner.host_fit_base(prof(10)) == [SWAP, SWAP, RECOMPUTE, SWAP]
    assert planner.host_fit_base(prof(9)) == [SWAP, RECOMPUTE, RECOMPUTE, SWAP]
    assert planner.host_fit_base(prof(3)) == [RECOMPUTE, RECOMPUTE, RECOMPUTE, KEEP]
    assert planner.host_fit_base(prof(0)) == [RECOMPUTE, RECOMPUTE, RECOMPUTE, KEEP]


# ---- shared host link (Reading 51), hand-traced on a 4-task DAG where a swap-in overlaps a
# swap-out. Tasks: F0 -> map 0; F1 reads 0 -> map 1; F2 reads 1 -> map 2; F3 reads 2 and 0 ->
# map 3 (sink). bwd(3) needs {2}, bwd(2) needs {1}, bwd(1) needs {0}. All fwd / bwd 10 ns;
# maps 0 and 1 swap (d2h 100 / 30, h2d 10 / 40), maps 2, 3 keep; unlimited memory.
#   F0 [0,10] F1 [10,20] F2 [20,30] F3 [30,40]; forward ends at 40.
#   O1 ready at 30 (last forward use F2): D2H [30, 60] alone. O0 ready at 40 (F3): waits for the lane.
#   At 60 O0 starts and I1 starts (eager: forward over, O1 done): both lanes busy.
#   Independent lanes (1000): I1 [60,100], O0 [60,160], I0 [160,170]; B3 [40,50], B2 [100,110],
#     B1 [170,180], B0 [180,190]: makespan 190.
#   duplex (500, 500): I1 needs 40 ns of work at 1/2 -> [60,140]; O0 has done 40 of 100 by 140,
#     the remaining 60 alone -> ends 200; I0 [200,210]; B2 [140,150], B1 [210,220], B0 [220,230]: 230.
#   duplex (800, 500): I1 [60,140] (O0 still running at 0.8: would need 125 ns); O0 has done
#     80 x 0.8 = 64 by 140, 36 alone -> 176; I0 [176,186]; B2 [140,150], B1 [186,196], B0 [196,206].
#   duplex (1000, 333): I1 work 40000 at 333 per ns -> ceil(40000 / 333) = 121 -> [60,181]; O0 at
#     full rate ends at 160 first, so at 160 I1 has 40000 - 100 x 333 = 6700 left, alone at 1000 per
#     ns -> ceil(6.7) = 7 -> ends 167; O0 [60,160]; I0 waits for the H2D lane: [167,177];
#     B2 [167,177], B1 [177,187], B0 [187,197]: 197.
def _link_dag(duplex):
    return Profile([10] * 4, [10] * 4, [1] * 4, [100, 30, 5, 5], [10, 40, 5, 5],
                   [[], [0], [1], [2, 0]], [[0], [0], [1], [2]], duplex=duplex)


@pytest.mark.parametrize("duplex,io,b,makespan", [
    ((1000, 1000), {"O1": (30, 60), "O0": (60, 160), "I1": (60, 100), "I0": (160, 170)},
     {3: (40, 50), 2: (100, 110), 1: (170, 180), 0: (180, 190)}, 190),
    ((500, 500), {"O1": (30, 60), "O0": (60, 200), "I1": (60, 140), "I0": (200, 210)},
     {2: (140, 150), 1: (210, 220), 0: (220, 230)}, 230),
    ((800, 500), {"O0": (60, 176), "I1": (60, 140), "I0": (176, 186)},
     {2: (140, 150), 1: (186, 196), 0: (196, 206)}, 206),
    ((1000, 333), {"O0": (60, 160), "I1": (60, 167), "I0": (167, 177)},
     {2: (167, 177), 1: (177, 187), 0: (187, 197)}, 197),
])
def test_shared_link_hand_trace(duplex, io, b, makespan):
    r = simulate(_link_dag(duplex), [SWAP, SWAP, KEEP, KEEP], EAGER)
    assert not r.oom
    got = {(k + str(m)): (s, e) for lane, k, m, s, e in r.events if lane != "COMPUTE"}
    for key, span in io.items():
        assert got[key] == span, key
    bw = {m: (s, e) for lane, k, m, s, e in r.events if lane == "COMPUTE" and k == "B"}
    for m, span in b.items():
        assert bw[m] == span, m
    assert r.makespan == makespan
