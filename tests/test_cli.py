"""The experiment driver keeps the reference CLI's interface (histostream/cli.py):
configuration precedence and source grammar on the CPU, and every mode end to end on
the GPU with the reference's CSV schemas."""
import json

import pytest

from paper_1011_0235_b200 import cli, datagen


def test_source_grammar():
    s = cli.parse_source("normal:100:5", 64, 3)
    assert (s.kind, s.mean, s.sigma, s.seed) == (datagen.NORMAL, 100.0, 5.0, 3)
    assert cli.parse_source("constant", 64, 0).value == 127
    m = cli.parse_source("mixture:0.6:9", 64, 0)
    assert (m.degeneracy, m.value) == (0.6, 9)
    assert cli.parse_source("random", 64, 0).kind == datagen.UNIFORM
    for bad in ("mixture", "file", "bogus:1", "normal:x"):
        with pytest.raises(cli.ConfigError):
            cli.parse_source(bad, 64, 0)
    segs = cli.parse_schedule("random@3,constant:1", 64, 0)
    assert [c for _, c in segs] == [3, None]
    with pytest.raises(cli.ConfigError):
        cli.parse_schedule(" , ", 64, 0)


def test_config_precedence(tmp_path):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"mode": "sweep", "seed": 4, "repetitions": 2}))
    run = cli.resolve_config(["--config", str(cfg), "--seed", "9"])
    assert (run.mode, run.seed, run.repetitions, run.slots) == ("sweep", 9, 2, 960)
    assert run.resolved_pixels() == 8192 * 8192 and run.out_path().name == "histostream_sweep.csv"
    cfg.write_text(json.dumps({"mode": "sweep", "bogus": 1}))
    with pytest.raises(cli.ConfigError):
        cli.resolve_config(["--config", str(cfg)])
    with pytest.raises(cli.ConfigError):
        cli.resolve_config([])
    assert cli.main([]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("mode,extra,header", [
    ("genealogy", [], "stage,throughput_bytes_per_sec"),
    ("compare", [], "distribution,kernel,throughput_bytes_per_sec,end_to_end_bytes_per_sec"),
    ("sweep", ["--source", "mixture:0.5:200"], "degeneracy,naive_tp,adaptive_tp,selected_kernel"),
    ("pipeline", ["--iterations", "6", "--window", "3"],
     "iteration,cpu_pre_us,transfer_in_us,compute_us,transfer_out_us,cpu_post_us,kernel_kind"),
    ("stream", ["--iterations", "8", "--window", "2", "--source", "random@4,constant:127"],
     "iteration,cpu_pre_us,transfer_in_us,compute_us,transfer_out_us,cpu_post_us,kernel_kind,degeneracy,divergence"),
])
def test_modes_on_gpu(cuda, tmp_path, mode, extra, header):
    out = tmp_path / f"{mode}.csv"
    dump = tmp_path / "pattern.txt"
    rc = cli.main(["--mode", mode, "--pixels", str(1 << 20), "--repetitions", "3", "--out", str(out),
                   "--pattern-dump", str(dump)] + extra)
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0] == header
    if mode == "compare":
        assert len(lines) == 11
    if mode == "sweep":
        assert len(lines) == 13 and lines[-1].startswith("crossover,")
    if mode == "stream":
        assert any(line.endswith("adaptive") or ",adaptive," in line for line in lines[1:])
    if mode != "compare":
        assert dump.read_text().strip()
