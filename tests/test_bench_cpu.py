"""bench.py helpers that run without a device: the ncu traffic lookup by kernel name
(profiles/traffic.json) and the argument surface the driver uses."""
import importlib.util
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_traffic_lookup_by_kernel_name():
    b = _bench()
    t5 = b.ncu_traffic(2, "k_pass1_big<5> (persistent step loop, row-layout copy, 16-byte paired columns)")
    t6 = b.ncu_traffic(2, "k_pass1_big<6> (persistent step loop, 16-byte paired columns)")
    assert t5 is not None and t6 is not None and t5 is not t6
    assert t5["kernel"] == "k_pass1_big<5>" and t6["kernel"] == "k_pass1_big<6>"
    for t in (t5, t6):
        assert t["dram_bytes_per_launch"] > t["algorithmic_bytes_per_launch"] > 0
        assert abs(t["ratio"] - t["dram_bytes_per_launch"] / t["algorithmic_bytes_per_launch"]) < 1e-9
    assert b.ncu_traffic(5, "k_stream_row2 (row, 16-byte paired columns)")["kernel"] == "k_stream_row2"


def test_cli_surface():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--e2e-concurrency"):
        assert flag in out.stdout
