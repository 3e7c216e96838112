"""Multi-rank host logic of the sharded build (distributed.py) on CPU: gloo process group,
world size 2 and 3, with an oracle-backed engine standing in for each rank's GPU.  The
assembled CSR must equal the reference golden CSR on every rank, and budget errors must be
raised identically everywhere."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleEngine:
    """Per-rank engine computing on the CPU oracle (test infrastructure only)."""

    def set_inputs(self, words, num_qubits, active, data, off, L, base, P, rows=None):
        from oracle.oracle import OracleInstance

        if rows is not None:
            self._r0 = rows[0]
        from paper_2401_06713_b200.driver import ColorLists

        n = active.size
        if off is None:
            lists = ColorLists.from_array(active, data.reshape(n, L), base, P)
        else:
            lists = ColorLists(active, [data[off[k]:off[k + 1]] for k in range(n)], base, P)
        self.inst = OracleInstance(words, active, lists, threads=2)
        self.csr = self.inst.build()
        self.n = n
        deg = np.zeros(n, dtype=np.int64)
        local = np.searchsorted(active, self.csr.members)
        deg[local] = np.diff(self.csr.offsets)
        self.deg = deg
        self.degu = self.csr.deg_upper
        # commuting partners j > i per row (row-wise K1 shard stand-in)
        w = words[active]
        self.comm_upper = np.zeros(n, dtype=np.int64)
        for i in range(n):
            acc = np.bitwise_xor.reduce(w[i + 1:] & w[i], axis=1) if i + 1 < n else np.zeros(0, np.uint64)
            self.comm_upper[i] = int((np.bitwise_count(acc) & 1 == 0).sum())

    def count(self, shard, nshards, r0, r1):
        a, b = self.n * shard // nshards, self.n * (shard + 1) // nshards
        rows = np.arange(a, b)
        pairs = int((self.n - 1 - rows).sum())
        return dict(anticommuting=pairs - int(self.comm_upper[a:b].sum()), pairs=pairs,
                    deg_sum=int(self.deg[r0:r1].sum()), members=int((self.deg[r0:r1] > 0).sum()))

    def degrees(self, rows):
        self.r = (self._r0, self._r0 + rows)
        return self.deg[self.r[0]:self.r[1]].astype(np.int32), self.degu[self.r[0]:self.r[1]].astype(np.int32)

    def fill_rows(self, gdeg, want):
        off = np.concatenate([[0], np.cumsum(np.asarray(gdeg, dtype=np.int64))])
        lo, hi = int(off[self.r[0]]), int(off[self.r[1]])
        return lo, hi, (self.csr.neighbors[lo:hi].copy() if want else None)


def _worker(rank, world, port, name, budget, two_phase, q, native=False, gather="root",
            exchange="auto"):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import GoldenCase
        from test_distributed import OracleEngine
        from paper_2401_06713_b200 import distributed as dmod
        from paper_2401_06713_b200.errors import EdgeBudgetExceededError
        import json

        with open(os.path.join(ROOT, "tests", "golden", "reference.json")) as f:
            meta = next(m for m in json.load(f)["cases"] if m["name"] == name)
        arrays = dict(np.load(os.path.join(ROOT, "tests", "golden", "builds_small.npz")))
        case = GoldenCase(meta, arrays)
        if native:
            eng = dmod.NativeEngine(0)
        else:
            eng = OracleEngine()
            eng._r0 = dmod.row_ranges(case.view.n_active, world)[rank][0]
        try:
            gc = dmod.build_sharded(case.view, case.lists, engine=eng, edge_budget=budget,
                                    two_phase=two_phase, gather=gather, exchange=exchange)
            if gather == "all" or rank == 0:
                case.check(gc)
            else:  # the header: everything but the neighbor ids
                assert gc.graph.neighbors.size == 0
                assert np.array_equal(gc.members, case.members)
                assert np.array_equal(gc.graph.offsets, case.offsets)
                assert gc.edge_count == case.meta["edge_count"]
                assert gc.view_edges_scanned == case.meta["view_edges_scanned"]
            q.put((rank, "ok", None))
        except EdgeBudgetExceededError as e:
            q.put((rank, "budget", e.projected))
    except Exception:  # report, don't hang the other ranks
        import traceback

        q.put((rank, "error", traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def _run(world, name, budget=None, two_phase=True, native=False, gather="root", target=None,
         args=None, exchange="auto"):
    # rank processes sharing one GPU: a transient CUDA initialisation failure of a freshly
    # spawned process (seen once on a box: "no usable CUDA device") is retried, not reported
    for attempt in range(3):
        out = _run_once(world, name, budget, two_phase, native, gather, target, args, exchange)
        if not (native and any(r[1] == "error" and "pcg_create" in str(r[2]) for r in out)):
            return out
    return out


def _run_once(world, name, budget, two_phase, native, gather, target, args, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    target = target or _worker
    args = args if args is not None else (name, budget, two_phase)
    extra = (native, gather, exchange) if target is _worker else (native, exchange)
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q, *extra))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out)


@pytest.mark.parametrize("world,name,gather", [(2, "tc_all_modes_pauli", "root"),
                                               (2, "ragged_lists", "all"),
                                               (3, "induced_subset", "root"),
                                               (3, "two_vertices", "all"),
                                               (3, "c1_iter1", "root")])
def test_sharded_build_matches_golden(world, name, gather):
    res = _run(world, name, gather=gather)
    assert [r[1] for r in res] == ["ok"] * world, res


def _run_worker(rank, world, port, name, q, native=False, exchange="auto"):
    """A whole sharded Picasso run (distributed.run_sharded) on one rank."""
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json

        import paper_2401_06713_b200 as b200
        from conftest import pauli_view, sha
        from test_distributed import OracleEngine
        from paper_2401_06713_b200 import distributed as dmod

        with open(os.path.join(ROOT, "tests", "golden", "reference.json")) as f:
            r = json.load(f)["runs"][name]
        v = pauli_view(r["n"], r["q"], r["gen_seed"])
        eng = dmod.NativeEngine(0) if native else OracleEngine()
        res = dmod.run_sharded(v, b200.PaletteParams(r["palette_pct"], r["alpha"], seed=r["seed"]),
                               strategy=r["strategy"], engine=eng, exchange=exchange)
        ok = (sha(res.color) == r["color_sha"] and res.total_colors == r["colors"]
              and len(res.iterations) == r["iterations"] and res.oracle_edges == r["oracle_edges"]
              and res.peak_conflict_edges == r["peak_conflict_edges"])
        q.put((rank, "ok" if ok else "mismatch", (sha(res.color), res.total_colors)))
    except Exception as e:  # report, don't hang the other ranks
        import traceback

        q.put((rank, "error", traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "c1"), (3, "tout_k3"), (2, "static_ldf")])
def test_sharded_whole_run_identical_coloring(world, name):
    """Algorithm 1 on N ranks (driver.py:272-385): every residue build sharded, the root colors
    and broadcasts; every rank ends with the reference's coloring."""
    res = _run(world, name, target=_run_worker, args=(name,))
    assert [r[1] for r in res] == ["ok"] * world, res


def test_sharded_budget_error_on_every_rank(golden_ref):
    meta = next(m for m in golden_ref["cases"] if m["name"] == "tc_determinism")
    res = _run(2, "tc_determinism", budget=meta["edge_count"] - 1)
    assert [r[1] for r in res] == ["budget", "budget"]
    assert res[0][2] == res[1][2] == meta["edge_count"]


def test_row_ranges_cover_rows():
    from paper_2401_06713_b200.distributed import row_ranges

    for n, w in ((0, 2), (1, 3), (10, 3), (1_000_003, 8)):
        rr = row_ranges(n, w)
        assert rr[0][0] == 0 and rr[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))


@pytest.mark.gpu
@pytest.mark.parametrize("world,name,gather,exchange",
                         [(2, "c1_iter1", "root", "p2p"), (2, "c1_iter1", "root", "collective"),
                          (3, "induced_subset", "all", "auto"), (2, "ragged_lists", "root", "p2p"),
                          (3, "tc_all_modes_pauli", "root", "p2p"), (3, "two_vertices", "root", "p2p")])
def test_sharded_native_engine_on_one_gpu(world, name, gather, exchange):
    """Each rank runs the CUDA K1 work-item shard + the owned masks of its rows + K2 row shard
    + sharded fill (all ranks share cuda:0); the root's CSR must equal the reference.  With
    exchange="p2p" every rank's fill stores its rows into the root's exported buffer (CUDA
    IPC between the rank processes, here on one device); "collective" gathers slices."""
    res = _run(world, name, native=True, gather=gather, exchange=exchange)
    assert [r[1] for r in res] == ["ok"] * world, res


@pytest.mark.gpu
@pytest.mark.parametrize("world,name,exchange", [(2, "c1", "p2p"), (3, "tout_k4", "p2p"),
                                                 (2, "c1", "collective")])
def test_sharded_whole_run_native_on_one_gpu(world, name, exchange):
    res = _run(world, name, native=True, target=_run_worker, args=(name,), exchange=exchange)
    assert [r[1] for r in res] == ["ok"] * world, res


@pytest.mark.gpu
def test_sharded_p2p_exchange_q32_20k_golden(golden_ref):
    """Three ranks on one GPU, peer-memory exchange: the root's CSR of the reference's
    20k-vertex q=32 build (hashes from the reference run) and the 4-byte id stores of three
    processes into one exported buffer."""
    res = _run(3, "q32_n20000", native=True, target=_p2p_worker, args=("q32_n20000",))
    assert [r[1] for r in res] == ["ok"] * 3, res


def _p2p_worker(rank, world, port, name, q, native=True, exchange="p2p"):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json

        from conftest import pauli_view, random_lists, sha
        from paper_2401_06713_b200 import distributed as dmod

        with open(os.path.join(ROOT, "tests", "golden", "reference.json")) as f:
            g = json.load(f)["builds_hashed"][name]
        v = pauli_view(20000, 32, 0)
        for _ in range(2):  # the second build reuses the exported buffer and the mappings
            gc = dmod.build_sharded(v, random_lists(v, seed=0), engine=dmod.NativeEngine(0),
                                    exchange=exchange)
            ok = sha(gc.graph.offsets) == g["offsets_sha"]
            if rank == 0:
                ok = ok and sha(gc.graph.neighbors) == g["neighbors_sha"]
            if not ok:
                break
        q.put((rank, "ok" if ok else "mismatch", None))
    except Exception:  # report, don't hang the other ranks
        import traceback

        q.put((rank, "error", traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_build_nccl_device_path(golden_ref):
    """build_sharded over NCCL (one rank): the slice is filled into a device buffer, gathered
    on the device and copied once into the pooled host buffer; the CSR must be the golden."""
    import os
    import subprocess
    import sys

    g = golden_ref["builds_hashed"]["q32_n20000"]
    code = (
        "import os, sys, hashlib, numpy as np, torch, torch.distributed as dist; "
        "sys.path.insert(0, 'tests'); "
        "import paper_2401_06713_b200 as b200; from paper_2401_06713_b200 import distributed as D; "
        "from conftest import pauli_view, random_lists; "
        "torch.cuda.set_device(0); dist.init_process_group('nccl'); "
        "v = pauli_view(20000, 32, 0); gc = D.build_sharded(v, random_lists(v, seed=0)); "
        "h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]; "
        "print(h(gc.graph.offsets), h(gc.graph.neighbors)); dist.destroy_process_group()"
    )
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split()[-2:] == [g["offsets_sha"], g["neighbors_sha"]]
