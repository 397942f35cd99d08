"""`cylspec` CLI (paper_2206_04827_b200/tools/ccf_cli.cpp, drop-in for proj/tools/cylspec_main.cpp):
the paths that end before any GPU work — configuration validation (runconfig.cpp:8-21), JSON config
parsing, CLI parse errors and the exit-code contract (0 ok, 2 config, 3 numerical / i/o;
cylspec_main.cpp:366-385)."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2206_04827_b200", "bin", "cylspec")


@pytest.fixture(scope="module")
def cli(P):
    if not os.path.exists(BIN):
        import __graft_entry__
        __graft_entry__.build()
    return BIN


def run(cli, *args, cwd=None):
    # never in the repo: the CLI writes failure_manifest.json under ./out on a failed run
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, cwd=cwd or tempfile.mkdtemp(),
                       timeout=120)
    return r.returncode, r.stderr


def test_exit_codes_without_gpu(cli, tmp_path):
    assert run(cli)[0] == 106  # a subcommand is required (CLI11 RequiredError)
    assert run(cli, "bogus")[0] == 109
    assert run(cli, "ns", "--m", "x")[0] == 104
    assert run(cli, "heat", "--wat", "1")[0] == 109
    rc, err = run(cli, "heat", "--bdf", "7")
    assert rc == 2 and "bdf_order must be 1..4" in err
    rc, err = run(cli, "heat", "--tol", "0.5")
    assert rc == 2 and "adi_tol" in err
    rc, err = run(cli, "transform")
    assert rc == 2 and "requires an input FieldFile" in err
    cfg = tmp_path / "c.json"
    cfg.write_text('{"m": 16, "n": 16, "p": 16, "steps": -1, "case": "decay"}')
    rc, err = run(cli, "heat", "--config", cfg)
    assert rc == 2 and "steps must be nonnegative" in err
    cfg.write_text('{"m": 16, "bc_kind": "robin"}')
    rc, err = run(cli, "heat", "--config", cfg)
    assert rc == 2 and "unknown bc kind" in err
    cfg.write_text('{"m": 16, ')
    rc, err = run(cli, "heat", "--config", cfg)
    assert rc == 2 and "config parse error" in err
    rc, err = run(cli, "heat", "--config", tmp_path / "none.json")
    assert rc == 2 and "cannot open config file" in err
    rc, err = run(cli, "transform", "--in", tmp_path / "missing.ccf", "--out", tmp_path / "o")
    assert rc == 3 and "i/o error" in err
    rc, err = run(cli, "bench", "--out", tmp_path / "o")
    assert rc == 2 and "outside the B200 hot path" in err
