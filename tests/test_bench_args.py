"""CPU: bench.py's device resolution (the --gpus path the driver's scaling
run takes) and its traffic lookup. No device needed."""
import json

import pytest

import bench


def test_single_process_uses_devices_0_to_n():
    assert bench.resolve_devices(1, 1, 8) == [0]
    assert bench.resolve_devices(4, 1, 8) == [0, 1, 2, 3]
    assert bench.resolve_devices(8, 1, 8) == list(range(8))


def test_more_gpus_than_visible_fails_loudly():
    with pytest.raises(SystemExit, match="only 1 sm_100 device"):
        bench.resolve_devices(2, 1, 1)
    with pytest.raises(SystemExit, match="must be >= 1"):
        bench.resolve_devices(0, 1, 1)


def test_torchrun_ranks_drive_their_local_device():
    assert bench.resolve_devices(4, 4, 8) is None
    with pytest.raises(SystemExit, match="one rank per GPU"):
        bench.resolve_devices(8, 4, 8)


def test_traffic_record_is_keyed_by_config_and_kernel(tmp_path, monkeypatch):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_traffic.json").write_text(json.dumps(
        {"c3:stripe_split_kernel": {"dram_bytes": 1024.0, "stripes": 512, "source": "x.ncu-rep"}}))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    assert bench.ncu_traffic("c3", "stripe_split_kernel")["stripes"] == 512
    assert bench.ncu_traffic("c2", "stripe_split_kernel") is None


def test_host_description_names_cpu_and_ram():
    h = bench.host_description()
    assert h["host_threads"] >= 1
    assert "cpu_model" in h and "ram_gib" in h
