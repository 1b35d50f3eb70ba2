"""The command line (paper_2009_07400_b200/__main__.py):
decks, presets, overrides, SimReport, XYZ trajectories."""

import json

import numpy as np
import pytest

from paper_2009_07400_b200.__main__ import (DeckError, _parse, format_report, parse_deck_text, read_xyz, resolve,
                                            write_xyz)


def test_preset_lj32_is_the_paper_configuration():
    cfg, opts = resolve(_parse(["--preset", "lj-32"]))
    assert cfg.unit_cells == (32, 32, 32) and cfg.n_atoms() == 131072 and cfg.steps == 100
    assert (cfg.dt, cfg.cutoff, cfg.verlet_buffer, cfg.reneigh_interval) == (0.005, 2.5, 0.3, 20)
    assert (cfg.epsilon, cfg.sigma, cfg.potential_kind) == (1.0, 1.0, "lj")
    assert opts["balance"] == "none" and opts["mode"] == "fast"


def test_preset_sd_halfdomain():
    cfg, _ = resolve(_parse(["--preset", "sd-halfdomain"]))
    assert cfg.potential_kind == "sd" and cfg.fill == "half-diagonal"
    assert cfg.stiffness == 0.0 and cfg.damping == 0.0 and cfg.steps == 1000
    assert cfg.diameter == cfg.cutoff == 1.2


def test_empty_deck_defaults_and_flag_precedence(tmp_path):
    assert parse_deck_text("") == {}
    deck = tmp_path / "run.deck"
    deck.write_text("# a comment\nunit_cells = 8 8 8\nsteps = 40\ndt=0.004\nranks = 2\ndump_every = 10\n")
    cfg, opts = resolve(_parse(["--preset", "lj-32", "--deck", str(deck), "--steps", "7", "--nz", "9"]))
    assert cfg.unit_cells == (8, 8, 9) and cfg.steps == 7 and cfg.dt == 0.004
    assert opts["ranks"] == 2 and opts["dump_every"] == 10


def test_deck_errors_name_line_and_field(tmp_path):
    with pytest.raises(DeckError, match="line 2: unknown key 'bogus'"):
        parse_deck_text("steps = 3\nbogus = 1\n")
    with pytest.raises(DeckError, match="line 1: bad value for dt: 'abc'"):
        parse_deck_text("dt = abc\n")
    with pytest.raises(DeckError, match="line 1: expected"):
        parse_deck_text("steps 3\n")
    with pytest.raises(Exception):
        resolve(_parse(["--nx", "1", "--ny", "1", "--nz", "1"]))  # domain smaller than r (core.py:247-252)
    with pytest.raises(DeckError, match="balancer"):
        resolve(_parse(["--balance", "hilbert"]))


def test_cli_sd_flags():
    cfg, _ = resolve(_parse(["--potential", "sd", "--damping", "0.5"]))
    assert cfg.potential_kind == "sd" and cfg.diameter == 1.2 and cfg.cutoff == 1.2 and cfg.damping == 0.5


def test_xyz_frames_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    st = np.hstack([rng.uniform(0, 5, (20, 3)), rng.normal(size=(20, 3))])
    p = tmp_path / "x.xyz"
    write_xyz(str(p), st, "Ar", "step 0")
    write_xyz(str(p), st[:4], "Ar", "step 5", append=True)
    frames = read_xyz(str(p))
    assert [c for c, _ in frames] == ["step 0", "step 5"]
    want = st[np.lexsort((st[:, 2], st[:, 1], st[:, 0]))][:, :3]
    assert np.array_equal(frames[0][1], want)  # %.17g round-trips fp64
    assert len(p.read_text().splitlines()) == 22 + 6


def test_report_is_key_value_lines():
    txt = format_report({"atoms": 4, "momentum_final": [0.0, 1.5, -2.0], "wall_s": 0.25})
    assert txt.splitlines() == ["atoms 4", "momentum_final 0.0 1.5 -2.0", "wall_s 0.25"]


@pytest.mark.gpu
def test_cli_runs_and_dumps_trajectory(tmp_path, capsys):
    """A 100-step run with --dump-every 20: 6 frames, the last the
    final state; the report's particle counts sum to the total; momentum drift
    within the acceptance bound."""
    from paper_2009_07400_b200.__main__ import main

    out = tmp_path / "traj.xyz"
    assert main(["--nx", "6", "--ny", "6", "--nz", "6", "--steps", "100", "--dump", str(out), "--dump-every", "20",
                 "--json"]) == 0
    rep = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    frames = read_xyz(str(out))
    assert [c.split()[-1] for c, _ in frames] == ["0", "20", "40", "60", "80", "100"]
    assert all(p.shape == (864, 3) for _, p in frames)
    assert rep["particles_rank_0"] == rep["atoms"] == 864 and rep["momentum_drift_max"] <= 1e-9


@pytest.mark.gpu
def test_cli_loopback_ranks_match_single_rank(tmp_path, capsys):
    """--ranks 4 without torchrun: four in-process ranks on one GPU; the final
    frame equals the single-rank run's within the parity tolerance and the
    per-rank counts sum to the total; --steps 0 is a report-only run."""
    from paper_2009_07400_b200.__main__ import main

    a, b = tmp_path / "a.xyz", tmp_path / "b.xyz"
    base = ["--nx", "8", "--ny", "8", "--nz", "8", "--steps", "30", "--json"]
    assert main(base + ["--dump", str(a)]) == 0
    capsys.readouterr()
    assert main(base + ["--ranks", "4", "--dump", str(b)]) == 0
    rep = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rep["ranks"] == 4 and sum(rep[f"particles_rank_{r}"] for r in range(4)) == 2048
    np.testing.assert_allclose(read_xyz(str(a))[-1][1], read_xyz(str(b))[-1][1], rtol=0, atol=1e-9)
    assert main(["--nx", "5", "--ny", "5", "--nz", "5", "--steps", "0", "--json"]) == 0
    assert json.loads(capsys.readouterr().out.strip().splitlines()[-1])["steps"] == 0


@pytest.mark.gpu
def test_cli_two_ranks(tmp_path):
    """torchrun + the CLI: 2 ranks over NCCL, rank 0 writes every atom."""
    import os
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "final.xyz"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                        "-m", "paper_2009_07400_b200", "--nx", "8", "--ny", "8", "--nz", "8", "--steps", "10",
                        "--json", "--dump", str(out)], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    assert out.read_text().splitlines()[0] == "2048"
