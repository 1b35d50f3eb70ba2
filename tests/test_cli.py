"""The command line wrapper (paper_2009_07400_b200/__main__.py)."""

import numpy as np
import pytest

from paper_2009_07400_b200.__main__ import _parse, config_from_args, write_xyz


def test_cli_config_defaults_and_sd():
    cfg = config_from_args(_parse(["--cells", "8", "8", "8", "--steps", "7"]))
    assert cfg.unit_cells == (8, 8, 8) and cfg.steps == 7 and cfg.cutoff == 2.5 and cfg.potential_kind == "lj"
    sd = config_from_args(_parse(["--potential", "sd", "--damping", "0.5"]))
    assert sd.potential_kind == "sd" and sd.diameter == 1.2 and sd.cutoff == 1.2 and sd.damping == 0.5
    with pytest.raises(Exception):
        config_from_args(_parse(["--cells", "1", "1", "1"]))  # domain smaller than r (core.py:247-252)


def test_xyz_dump_sorted_exact(tmp_path):
    rng = np.random.default_rng(0)
    st = np.hstack([rng.uniform(0, 5, (20, 3)), rng.normal(size=(20, 3))])
    p = tmp_path / "x.xyz"
    write_xyz(str(p), st, "Ar", "test")
    lines = p.read_text().splitlines()
    assert lines[0] == "20" and lines[1] == "test"
    got = np.array([[float(v) for v in ln.split()[1:]] for ln in lines[2:]])
    want = st[np.lexsort((st[:, 2], st[:, 1], st[:, 0]))][:, :3]
    assert np.array_equal(got, want)  # %.17g round-trips fp64


@pytest.mark.gpu
def test_cli_runs_and_dumps(tmp_path, capsys):
    from paper_2009_07400_b200.__main__ import main

    out = tmp_path / "final.xyz"
    assert main(["--cells", "5", "5", "5", "--steps", "6", "--thermo-every", "3", "--dump", str(out)]) == 0
    text = capsys.readouterr().out
    assert "atom-steps/s" in text
    assert out.read_text().splitlines()[0] == "500"


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
                        "-m", "paper_2009_07400_b200", "--cells", "8", "8", "8", "--steps", "10", "--json",
                        "--dump", str(out)], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    assert out.read_text().splitlines()[0] == "2048"
