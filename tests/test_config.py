"""load_config, the CSV writers and the
CLI's usage contract — host code, no GPU."""
import csv

import numpy as np
import pytest

from paper_2206_05761_b200 import config, io
from paper_2206_05761_b200.abi import BAND_PARENTS, BC_TRANSMISSIVE

MINIMAL = """
[case]
name = circular
[grid]
L = 8
epsilon = 1e-3
[time]
t_end = 3.5
"""


def test_minimal_config_defaults_filled():
    rc = config.parse_config(MINIMAL)  # SPEC.md:561 "minimal config ... valid, defaults filled"
    assert rc.get("grid.L") == 8 and rc.get("physics.cfl") == 0.5 and rc.get("physics.h_dry") == 1e-6
    cfg, h, qx, qy, z = config.build_state(rc)
    assert cfg.L == 8 and cfg.epsilon == 1e-3 and cfg.t_end == 3.5 and h.shape == (256, 256)


@pytest.mark.parametrize("bad,where,what", [
    (MINIMAL.replace("epsilon = 1e-3", "epsilon = -1"), "grid.epsilon", ">= 0"),
    (MINIMAL.replace("L = 8", "L = 20"), "grid.L", "outside [1, 13]"),
    (MINIMAL + "[grid]\nepsilom = 1\n", "<config>:10:1", "unknown key grid.epsilom"),  # no silent typos
    (MINIMAL + "[gird]\n", "<config>:9:1", "unknown section"),
    (MINIMAL + "[time]\n  t_end 3\n", "<config>:10:3", "expected key = value"),
    (MINIMAL.replace("L = 8", "L = eight"), "<config>:5:1", "invalid int"),
    (MINIMAL.replace("name = circular", "name = tsunami"), "<config>:3:1", "unknown case"),
    ("L = 3\n", "<config>:1:1", "before any [section]"),
    ("[case]\nname = circular\n", "grid.L", "required"),
])
def test_config_errors_are_located(bad, where, what):
    with pytest.raises(config.ConfigError) as e:
        config.parse_config(bad)
    assert e.value.where.startswith(where) and what in str(e.value), str(e.value)


def test_overrides_and_sections():
    rc = config.parse_config(MINIMAL + "[boundary]\nwest = transmissive\n[output]\ngauges = a 1 2; b -3 4.5\n",
                             overrides=["grid.L=6", "grid.band=parents", "time.output_times=1,2"])
    cfg, *_ = config.build_state(rc)
    assert cfg.L == 6 and cfg.band_mode == BAND_PARENTS and cfg.bc[0] == BC_TRANSMISSIVE
    assert tuple(cfg.output_times) == (1.0, 2.0)
    assert rc.get("output.gauges") == (("a", 1.0, 2.0), ("b", -3.0, 4.5))
    with pytest.raises(config.ConfigError):
        config.parse_config(MINIMAL, overrides=["grid.LL=3"])
    with pytest.raises(config.ConfigError):
        config.parse_config(MINIMAL, overrides=["time.output_times=2,1"])


def test_config_parsing_is_total():
    """Fuzz: every input yields a RunConfig or a ConfigError."""
    rng = np.random.default_rng(3)
    alphabet = list("[]=#.,; \n-+eE0123456789abcdefghijklmnopqrstuvwxyzL_")
    for _ in range(400):
        text = "".join(rng.choice(alphabet, size=int(rng.integers(0, 80))))
        try:
            config.parse_config(MINIMAL + text)
        except config.ConfigError:
            pass


def test_gauge_and_step_csv(tmp_path):
    p = tmp_path / "g.csv"
    io.write_gauges(p, [], [], names=[])  # empty gauge list -> header-only file
    assert p.read_text() == "t\n"
    vals = [np.arange(8.0).reshape(4, 2) + k for k in range(3)]
    io.write_gauges(p, [0.0, 0.5, 1.0], vals, names=["west", "east"])
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["t", "west_h", "west_qx", "west_qy", "west_eta", "east_h", "east_qx", "east_qy", "east_eta"]
    assert [float(x) for x in rows[2]] == [0.5, 1, 3, 5, 7, 2, 4, 6, 8]
    rep = {"step": 3, "t": 0.1 + 0.2, "dt": 1e-3, "dt_used": 2e-3, "n_leaves": 4096, "n_leaves_next": 4096,
           "ms_encode_flag": 0.0, "ms_band_closure": 0.0, "ms_decode_traverse": 0.0, "ms_neighbours": 0.0,
           "ms_fv1": 0.0, "ms_total": 0.0, "n_near_threshold": 0}
    s = tmp_path / "s.csv"
    io.write_step_reports(s, [rep])
    io.write_step_reports(s, [dict(rep, step=4)], append=True)
    rows = list(csv.DictReader(open(s)))
    assert [r["step"] for r in rows] == ["3", "4"] and float(rows[0]["t"]) == 0.1 + 0.2  # 17 digits: exact
    assert rows[0]["n_leaves"] == "4096"  # eps = 0 column constant 4^L


def test_cli_usage_errors(tmp_path, capsys):
    from paper_2206_05761_b200 import cli

    assert cli.main([]) == 2  # no subcommand: usage
    assert cli.main(["run"]) == 2  # missing config: exit 2
    assert cli.main(["run", "--config", str(tmp_path / "nope.cfg")]) == 2
    bad = tmp_path / "bad.cfg"
    bad.write_text(MINIMAL.replace("L = 8", "L = 20"))
    assert cli.main(["run", "--config", str(bad)]) == 2
    assert "grid.L" in capsys.readouterr().err
    assert cli.main(["validate", "--only", "A99"]) == 2
    assert cli.main(["compare", str(tmp_path / "x"), str(tmp_path / "y")]) == 2
