"""ScoutEngine scheduler contract on the host (no GPU): the reference's
scheduler criterion (test_acceptance.py:372-441) run against the drop-in --
dequeue order equals the sort oracle over 1,024 random priorities, 10,000
fuzzed scheduler events keep stages monotone and eviction always lands
within budget -- plus tile candidates ordered after patches of equal
priority (engine.py:218-242)."""
import threading

import numpy as np

from paper_2509_20198_b200.engine import (EngineConfig, PatchState, ScoutEngine,
                                          Stage, TileResidency, TileState)
from paper_2509_20198_b200.patches import patch_grid_for
from paper_2509_20198_b200.refiner import WeightBundle, identity_descriptor


def _fake(ni=32, nj=32):
    class _Box:
        pass
    ds = _Box()
    ds.tiles = []
    ds.bbox_min = np.array([0.0, 0.0, 0.0])
    ds.bbox_max = np.array([ni * 640.0, nj * 640.0, 100.0])
    eng = ScoutEngine.__new__(ScoutEngine)
    eng.dataset = ds
    eng.config = EngineConfig()
    eng.weights = WeightBundle(1, {}, identity_descriptor())
    eng._identity = eng.weights
    eng.grid = patch_grid_for(ds.bbox_min, ds.bbox_max)
    eng.patches = {(k.i, k.j): PatchState(key=k, stage=Stage.CHUNK_POINTS_ONLY)
                   for k in eng.grid.keys()}
    eng.tiles = {}
    eng.raw, eng.refined, eng.resident_records, eng.pending_bakes = {}, {}, {}, {}
    eng.frame = 0
    eng.chunk_points_loaded = eng.chunk_points_expected = 0
    eng.ready_events = []
    eng.lock = threading.RLock()
    eng._tile_by_id = {}
    return eng


def test_dequeue_matches_sort_oracle():
    rng = np.random.default_rng(2024)
    eng = _fake(32, 32)
    prios = rng.random(len(eng.patches)) * 1e6
    prios[::7] = prios[0]  # ties resolve by patch id
    for p, state in zip(prios, eng.patches.values()):
        state.priority = float(p)
    tasks = eng.next_tasks(len(eng.patches))
    expect = sorted(eng.patches, key=lambda pid: (-eng.patches[pid].priority, pid))
    assert [t.patch for t in tasks] == expect
    assert all(s.in_flight for s in eng.patches.values())
    assert eng.next_tasks(5) == []


def test_tiles_after_patches_of_equal_priority():
    eng = _fake(2, 2)
    for s in eng.patches.values():
        s.priority = 5.0
    eng.tiles = {3: TileResidency(tile_id=3, priority=5.0, wanted=True),
                 1: TileResidency(tile_id=1, priority=9.0, wanted=True)}
    kinds = [(t.kind, t.patch or t.tile_id) for t in eng.next_tasks(10)]
    assert kinds[0] == ("load_tile", 1)
    assert kinds[-1] == ("load_tile", 3)
    assert eng.tiles[1].state == TileState.LOADING


def test_fuzzed_events_monotone_and_budget_safe():
    rng = np.random.default_rng(2024)
    eng = _fake(8, 8)
    for tid in range(16):
        eng.tiles[tid] = TileResidency(tile_id=tid)
    last = {pid: s.stage for pid, s in eng.patches.items()}
    events, in_flight = 0, []
    while events < 10_000:
        op = int(rng.integers(0, 10))
        if op == 0:
            for state in eng.patches.values():
                state.priority = float(rng.random())
        elif op == 1:
            for tid, res in eng.tiles.items():
                if res.state == TileState.COLD and rng.random() < 0.2:
                    res.state = TileState.RESIDENT
                    res.memory_bytes = int(rng.integers(1, 100)) * 1024
                    eng.resident_records[tid] = np.zeros(2)
            budget = int(rng.integers(0, 3_000_000))
            eng.evict(budget)
            resident = sum(r.memory_bytes for r in eng.tiles.values()
                           if r.state == TileState.RESIDENT)
            assert resident <= budget
        else:
            in_flight.extend(eng.next_tasks(int(rng.integers(1, 6))))
            rng.shuffle(in_flight)
            take = in_flight[:max(1, len(in_flight) // 2)]
            in_flight = in_flight[len(take):]
            for task in take:
                st = eng.patches[task.patch]
                st.in_flight = False
                if task.kind == "interpolate":
                    eng.raw[task.patch] = "raw"
                    eng._advance(st, Stage.INTERPOLATED)
                elif task.kind == "refine":
                    eng._advance(st, Stage.REFINED)
                events += 1
        for pid, state in eng.patches.items():
            assert state.stage >= last[pid], "stage regressed"
            last[pid] = state.stage
        events += 1


def test_patch_table_views_stay_consistent():
    """PatchState attributes read and write the engine's patch table once it
    exists (structure of arrays behind the reference API): values set before
    the table is built are kept, later writes through either side agree,
    and replacing the patch dict rebuilds the table."""
    eng = _fake(4, 4)
    pids = list(eng.patches)
    eng.patches[pids[3]].priority = 7.5
    eng.patches[pids[5]].no_data = True
    t = eng._table()
    assert t.priority[3] == 7.5 and bool(t.no_data[5])
    st = eng.patches[pids[6]]
    st.stage = Stage.REFINED
    assert t.stage[6] == Stage.REFINED and st.stage is Stage.REFINED
    t.in_flight[7] = True
    assert eng.patches[pids[7]].in_flight is True
    assert eng.progress()["refined"] == 1 / 16
    tasks = eng.next_tasks(100)
    assert all(t_.patch not in (pids[5], pids[6], pids[7]) for t_ in tasks)
    assert len(tasks) == 13
    eng.patches = {p: PatchState(key=eng.grid.key(*p), stage=Stage.CHUNK_POINTS_ONLY)
                   for p in pids}
    assert len(eng.next_tasks(100)) == 16  # fresh states: a fresh table
