"""bench.py's reference arm on CPU (the oracle on a bounded sample): one JSON line with the
contract's keys; under torchrun only rank 0 prints (other ranks exit 0 without work)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--ref-sample", "65536"], capture_output=True, text=True, env=env,
                       cwd=REPO, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


def test_reference_arm_other_ranks_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


def test_multi_gpu_line_contract():
    """The N > 1 JSON line (bench.multi_line, fed synthetic measurements): contract keys, cfg5
    shapes (2^33 strong headline, int64), value = all ranks' keys / max-over-ranks time."""
    sys.path.insert(0, REPO)
    import bench
    for world in (2, 4, 8):
        shapes = bench.multi_shapes(world)
        head = shapes[0]
        assert head[1] == "strong" and head[2] == "i64" and head[3] * world == 1 << 33
        assert {s[0] for s in shapes} == {"strong_i64", "strong_f64", "weak_i64", "weak_f64"}
        results = {nm: {"ms": 100.0, "mode": md, "dtype": dt, "n_per_rank": nl, "a2a_ms": 10.0,
                        "a2a_bytes": nl * 8 * (world - 1) // world, "n_out": nl, "pass_ms": 5.0,
                        "pass_bytes": 2 * nl * 8} for nm, md, dt, nl in shapes}
        d = bench.multi_line(world, 5, 3, head, results, {"ms": 200.0, "h2d": head[3] * 8, "d2h": head[3] * 8},
                             700.0, 123, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []})
        json.dumps(d)
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                  "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                  "gpu_launches", "clocks"):
            assert k in d, k
        assert d["n_gpus"] == world and d["scaling"] == "strong" and d["dtype"] == "i64"
        assert abs(d["value"] - (1 << 33) / 0.1) < 1e-6 * d["value"]
        assert d["e2e"]["h2d_bytes_per_step"] == head[3] * 8 and d["e2e"]["value"] < d["value"]
        rf = d["roofline"]
        assert rf["bound"] == "hbm" and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
        assert rf["a2a"]["nccl_all_to_all_1GiB_pair_GBps"] == 700.0
        assert set(d["configs"]) == {s[0] for s in shapes}
    # one GPU (--force-dist): the weak shape is the headline (2^33 keys do not fit one GPU)
    assert bench.multi_shapes(1)[0] == ("weak_i64", "weak", "i64", 1 << 30)
