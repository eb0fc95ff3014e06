"""CLI contract (reference cli.py): config parsing and hash
against the reference's own (tests/golden/cli.npz), exit codes; the device
runs of train / bench-insertion / bench-samplers write the reference's CSVs."""

import dataclasses
import os

import numpy as np
import pytest

from paper_1903_03129_b200 import cli
from tests.golden.make_golden_data import CLI_TOML, XC_GOOD


def _toml(tmp_path, text=CLI_TOML):
    p = tmp_path / "run.toml"
    p.write_text(text)
    return str(p)


def test_config_fields_and_hash_equal_the_reference(golden, tmp_path):
    g = golden("cli")
    assert [f.name for f in dataclasses.fields(cli.RunConfig)] == g["fields"].tolist()
    assert cli.config_hash(cli.RunConfig()) == g["hash_default"][0]
    cfg = cli.load_config(_toml(tmp_path))
    assert cli.config_hash(cfg) == g["hash"][0]
    assert cfg.beta == g["beta"][0] and cfg.hidden == g["hidden"].tolist()


def test_config_errors_exit_2(tmp_path, capsys):
    assert cli.main(["train", "--config", _toml(tmp_path, "[model]\nbogus = 1\n")]) == 2
    assert "unknown config key model.bogus" in capsys.readouterr().err
    assert cli.main(["train", "--config", _toml(tmp_path, "[weird]\nk = 1\n")]) == 2
    assert cli.main(["train", "--config", _toml(tmp_path)]) == 2  # train.txt does not exist
    assert "train file not found" in capsys.readouterr().err
    assert cli.main(["bench-samplers", "--config", _toml(tmp_path), "--workers", "0"]) == 2


def test_csv_starts_with_config_hash(tmp_path):
    cfg = cli.load_config(_toml(tmp_path))
    path = cli.write_csv(tmp_path / "x.csv", cfg, ["a", "b"], [(1, 2.5)])
    lines = path.read_text().splitlines()
    assert lines == [f"# config-hash: {cli.config_hash(cfg)}", "a,b", "1,2.5"]


@pytest.mark.gpu
def test_device_commands_write_reference_csvs(tmp_path):
    from paper_1903_03129_b200.data import CorpusSpec, Dataset, save_xc_file, synthetic_corpus

    spec = CorpusSpec(500, 300, ("uniform", 5, 20), 1.1, ("uniform", 1, 3), 1.1, False)
    c = synthetic_corpus(spec, 200, seed=1)
    save_xc_file(Dataset([c.example(i) for i in range(len(c))], 500, 300), tmp_path / "train.txt")
    toml = CLI_TOML.replace('train = "train.txt"', f'train = "{tmp_path / "train.txt"}"')
    out = tmp_path / "out"
    assert cli.main(["train", "--config", _toml(tmp_path, toml), "--out", str(out)]) == 0
    lines = (out / "train_log.csv").read_text().splitlines()
    assert lines[0].startswith("# config-hash: ")
    assert lines[1] == "iteration,wall_seconds,train_loss,test_P@1,test_P@5,mean_active_fraction_per_lsh_layer"
    its = [int(r.split(",")[0]) for r in lines[2:]]
    assert its == [5, 10, 14]  # 2 epochs x ceil(200 / 32) = 14 iterations, every 5, then the tail
    assert (out / "final.ckpt").read_bytes()[:4] == b"SLDE"
    for cmd, name, header in (("bench-insertion", "bench_insertion.csv",
                               "policy,insert_to_ht_seconds,full_insertion_seconds"),
                              ("bench-samplers", "bench_samplers.csv", "strategy,n,seconds")):
        assert cli.main([cmd, "--config", _toml(tmp_path, toml), "--out", str(out)]) == 0
        assert (out / name).read_text().splitlines()[1] == header
