"""CPU-side checks: the C-ABI library loads and exports its header, host logic
(config validation, decomposition, lattice) matches the oracle bit for bit."""

import os

import numpy as np
import pytest

import oracle as O
import paper_2009_07400_b200 as P
from paper_2009_07400_b200 import _native as N


def test_library_exports_every_header_symbol():
    syms = N.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(N.lib, s)]
    assert not missing
    assert N.lib.tmd_version() == 1
    assert N.launch_count() >= 0


def test_step_run_struct_layout_matches_header(tmp_path):
    """N.StepRun (ctypes) has TmdStepRun's size and field offsets (gcc on the header)."""
    import ctypes
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    fields = [f for f, _ in N.StepRun._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "tinymd_b200.h"\nint main(void){\n'
                   + 'printf("%zu\\n", sizeof(TmdStepRun));\n'
                   + "".join(f'printf("%zu\\n", offsetof(TmdStepRun, {f}));\n' for f in fields) + "return 0;}\n")
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(N.StepRun)
    assert got[1:] == [getattr(N.StepRun, f).offset for f in fields]


def test_epoch_struct_layout_matches_header(tmp_path):
    """N.EpochP1 (ctypes) has TmdEpochP1's size and field offsets."""
    import ctypes
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    fields = [f for f, _ in N.EpochP1._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "tinymd_b200.h"\nint main(void){\n'
                   + 'printf("%zu\\n", sizeof(TmdEpochP1));\n'
                   + "".join(f'printf("%zu\\n", offsetof(TmdEpochP1, {f}));\n' for f in fields) + "return 0;}\n")
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(N.EpochP1)
    assert got[1:] == [getattr(N.EpochP1, f).offset for f in fields]


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(ln.split(".")[-2] for ln in out.stdout.split() if ln.endswith(".cubin"))
    assert archs == {"sm_100a"}, archs


@pytest.mark.parametrize("bad", [
    dict(unit_cells=(0, 4, 4)), dict(particles_per_cell=3), dict(cutoff=0.0), dict(verlet_buffer=-1.0),
    dict(steps=-1), dict(reneigh_interval=0), dict(potential_kind="eam"), dict(layout_kind="xyz"),
    dict(layout_kind="aosoa", aosoa_cluster=3), dict(fill="some"), dict(unit_cells=(1, 1, 1)),
])
def test_config_rejections(bad):
    # test_core.py:137-153
    with pytest.raises(P.ConfigError):
        P.SimConfig(**bad).validate()


def test_config_derived_quantities():
    cfg = P.SimConfig().validate()
    assert cfg.interaction_radius() == 2.8
    assert cfg.lattice_constant() == (4 / 0.8442) ** (1.0 / 3.0)
    assert np.array_equal(cfg.domain().hi, O.domain_bounds(cfg)[1])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6, 8, 12, 16])
def test_decomposition_matches_oracle(p):
    cfg = P.SimConfig(unit_cells=(12, 12, 12))
    lo, hi = O.domain_bounds(cfg)
    assert P.factor_rank_grid(p) == O.factor_rank_grid(p)
    for rank in range(p):
        d = P.Decomposition(cfg.domain(), p, rank, 2.8)
        rounds, slab = O.stencil_entries(O.factor_rank_grid(p), rank, lo, hi)
        assert np.array_equal(d.slab.lo, slab[0]) and np.array_equal(d.slab.hi, slab[1])
        for mine, theirs in zip(d.rounds, rounds):
            for a, b in zip(mine, theirs):
                assert (a.dim, a.sign, a.send_to, a.recv_from, a.face) == (b.dim, b.sign, b.send_to,
                                                                        b.recv_from, b.face)
                assert np.array_equal(a.shift, b.shift)


def test_factor_rank_grid_known():
    assert [P.factor_rank_grid(p) for p in (1, 2, 4, 8)] == [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]


@pytest.mark.parametrize("cells,fill", [((8, 8, 8), "full"), ((5, 7, 3), "full"), ((6, 6, 6), "half-diagonal")])
def test_lattice_bitwise_vs_oracle(cells, fill):
    cfg = P.SimConfig(unit_cells=cells, fill=fill)
    pos = P.lattice_positions(cfg, cfg.domain())
    vel = P.lattice_velocities(cfg, pos.shape[0])
    op, ov = O.initial_state(cfg)
    assert np.array_equal(pos, op) and np.array_equal(vel, ov)


def test_pbc_and_minimum_image():
    # test_core.py:20-87
    box = P.AABB.cube(0.0, 10.0)
    p = np.array([[10.0, -0.5, 25.0], [3.0, 4.0, 5.0]])
    w = P.pbc_correct(p, box)
    assert np.all((w >= 0.0) & (w < 10.0))
    assert np.array_equal(w[1], p[1])
    assert np.array_equal(P.pbc_correct(w, box), w)
    d = P.minimum_image(np.array([[6.0, -6.0, 4.0]]), box)
    assert np.allclose(d, [[-4.0, 4.0, 4.0]])
