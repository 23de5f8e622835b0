"""The C++ drop-in (the reference's tools/txsite_main.cpp + txsite_core, proj/
CMakeLists.txt:13-28) on the B200: the txsite CLI with SPEC.md:468's flags plus
the BASELINE additions (--water-rows, --observers-random, --gpus/--devices,
--exchange), its artefacts (result CSV SPEC.md:412, report SPEC.md:428, dumps
SPEC.md:201,262,331), load_binary, and the C++ value-type API
(txsite::estimate_vix(grid, ...) ... site(viewsheds, ...)) -- each against the
CPU oracle or the Python path."""
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2006_16783_b200", "bin", "txsite")
API = os.path.join(ROOT, "paper_2006_16783_b200", "bin", "txsite_api_check")


def _run(args, d, ok=True):
    r = subprocess.run([EXE] + [str(a) for a in args] + ["--out-dir", str(d)], capture_output=True, text=True,
                       timeout=900)
    if ok:
        assert r.returncode == 0, r.stderr
    return r


def _csv(d):
    lines = (d / "result.csv").read_text().strip().splitlines()
    assert lines[0] == "rank,row,col,marginal_gain,cumulative_coverage"
    return [tuple(l.split(",")) for l in lines[1:]]


def _oracle(z, roi, ht, hr, S, bw, k, target, max_sel, vseed, observers=None):
    nr, nc = z.shape
    if observers:
        rows, cols = O.random_observers(nr, nc, *observers)
        vix, sc = None, np.zeros(len(rows), np.int32)
    else:
        vix = O.estimate_vix(z, roi, ht, hr, S, vseed)
        rows, cols, sc = O.find_candidates(vix, bw, k)
    wins, words = O.viewsheds(z, roi, ht, hr, rows, cols)
    o = O.site(rows, cols, wins, words, nr, nc, target, max_selected=max_sel)
    return o, vix, (rows, cols, sc), (wins, words)


def _check_csv(rows, o, nr, nc):
    got = [(int(r), int(c), int(g)) for _, r, c, g, _ in rows]
    assert got == list(zip(o["row"].tolist(), o["col"].tolist(), o["gain"].tolist()))
    assert [float(x[4]) for x in rows] == o["coverage"].tolist()


BASE = ["--synth", "--nrows", 320, "--ncols", 288, "--seed", 9, "--roughness", 0.55, "--roi", 24,
        "--tx-height", 12, "--rx-height", 6, "--samples", 8, "--per-block", 3, "--block-width", 32,
        "--coverage", 0.95, "--max-selected", 60, "--vix-seed", 4]


@pytest.mark.parametrize("devices", [None, "0,0", "0,0,0"])
def test_cli_water_rows_dumps_and_group(tmp_path, devices):
    """Config-3 style water clamp, all three dumps, single context and the
    native group (row bands on virtual ranks, P2P exchange)."""
    args = BASE + ["--water-rows", 40, "--dump-vix", "--dump-candidates", "--dump-viewsheds", "--snapshots", "1,8"]
    if devices:
        args += ["--devices", devices]
    _run(args, tmp_path)
    z = O.generate_fractal(320, 288, 0.55, 9, 0, 4000)
    z[:40] = 0
    o, vix, (rows, cols, sc), (wins, words) = _oracle(z, 24, 12, 6, 8, 32, 3, 0.95, 60, 4)
    _check_csv(_csv(tmp_path), o, 320, 288)
    pgm = (tmp_path / "cumshed.pgm").read_bytes()
    hdr = b"P5\n288 320\n255\n"
    img = np.frombuffer(pgm[len(hdr):], np.uint8).reshape(320, 288)
    assert np.array_equal(img == 255, O.dense_bits(o["cum"], 320, 288) == 1)
    assert np.array_equal(np.fromfile(tmp_path / "vix.u8", np.uint8).reshape(320, 288), vix)
    cl = (tmp_path / "candidates.csv").read_text().strip().splitlines()
    assert cl[0] == "row,col,score"
    assert [tuple(map(int, l.split(","))) for l in cl[1:]] == list(zip(rows.tolist(), cols.tolist(), sc.tolist()))
    raw = (tmp_path / "viewsheds.bin").read_bytes()
    off = 0
    for i in range(len(rows)):
        r0, c0, w, h = np.frombuffer(raw, np.int32, 4, off)
        off += 16
        nw = (int(h) * int(w) + 63) // 64
        v = np.frombuffer(raw, np.uint64, nw, off)
        off += 8 * nw
        assert (r0, c0, h, w) == tuple(wins[i]) and np.array_equal(v, words[i][:nw]), i
    assert off == len(raw)
    s8 = np.frombuffer((tmp_path / "cumshed_8.pgm").read_bytes()[len(hdr):], np.uint8)
    s1 = np.frombuffer((tmp_path / "cumshed_1.pgm").read_bytes()[len(hdr):], np.uint8)
    assert (s1 <= s8).all() and (s8 <= img.reshape(-1)).all()
    rep = (tmp_path / "report.txt").read_text()
    assert "peak_memory_estimate device_bytes=" in rep and "params input=synth nrows=320" in rep
    assert f"gpus={len(devices.split(',')) if devices else 1}" in rep


@pytest.mark.parametrize("devices", [None, "0,0"])
def test_cli_random_observers(tmp_path, devices):
    """Config-5 style: random observers replace VIX + FINDMAX."""
    args = ["--synth", "--nrows", 300, "--ncols", 260, "--seed", 2, "--roi", 30, "--tx-height", 50,
            "--rx-height", 50, "--coverage", 1.0, "--max-selected", 80, "--observers-random", 2500,
            "--observer-seed", 31, "--block-width", 50, "--no-images"]
    if devices:
        args += ["--devices", devices]
    _run(args, tmp_path)
    z = O.generate_fractal(300, 260, 0.5, 2, 0, 4000)
    o, *_ = _oracle(z, 30, 50, 50, 0, 0, 0, 1.0, 80, 0, observers=(2500, 31))
    _check_csv(_csv(tmp_path), o, 300, 260)
    assert not (tmp_path / "cumshed.pgm").exists()


def test_cli_exchanges_agree(tmp_path):
    outs = []
    for k, extra in enumerate([[], ["--devices", "0,0", "--exchange", "host"], ["--devices", "0,0,0,0"],
                               ["--devices", "0,0,0", "--exchange", "p2p"], ["--gpus", "1", "--exchange", "nccl"]]):
        d = tmp_path / f"r{k}"
        d.mkdir()
        _run(BASE + extra + ["--no-images"], d)
        outs.append((d / "result.csv").read_bytes())
    assert all(x == outs[0] for x in outs)


def test_cli_load_binary(tmp_path):
    """--input of raw int16 LE: same result as the synthetic run;
    a size mismatch and the NODATA sentinel abort with stage-tagged messages."""
    z = O.generate_fractal(320, 288, 0.55, 9, 0, 4000)
    f = tmp_path / "t.bin"
    z.astype("<i2").tofile(f)
    a, b = tmp_path / "a", tmp_path / "b"
    a.mkdir(); b.mkdir()
    _run(BASE, a)
    args = [x if x != "--synth" else "--input" for x in BASE]
    args.insert(args.index("--input") + 1, str(f))
    _run(args, b)
    assert (a / "result.csv").read_bytes() == (b / "result.csv").read_bytes()
    bad = [str(x) for x in args]
    bad[bad.index("--ncols") + 1] = "287"
    r = _run(bad, tmp_path, ok=False)
    assert r.returncode == 1 and "[read] size-mismatch" in r.stderr
    z2 = z.copy()
    z2[5, 5] = -32768
    z2.astype("<i2").tofile(f)
    r = _run(args, tmp_path, ok=False)
    assert r.returncode == 1 and "NODATA" in r.stderr


def test_cpp_value_type_api(tmp_path):
    r = subprocess.run([API, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    out = {l.split(" ", 1)[0]: l.split(" ", 1)[1] for l in r.stdout.strip().splitlines()}
    z = O.generate_fractal(160, 140, 0.5, 3, 0, 2000)
    assert out["roundtrip"] == "1"
    assert out["size_mismatch"].startswith("7 ") and "size-mismatch" in out["size_mismatch"]
    assert float(out["elev"]) == O.elevation_between(int(z[10, 10]), int(z[10, 11]), 1, 4)
    v1 = O.is_visible(z, 20, 30, 10, 60, 90, 5)
    v2 = O.is_visible(z, 100, 20, 0, 101, 21, 0)
    assert out["visible"] == f"{int(v1)} {int(v2)}"
    vix = O.estimate_vix(z, 15, 10, 5, 7, 11)
    h = 1469598103934665603
    for s in vix.reshape(-1).tolist():
        h = ((h ^ s) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    assert int(out["vix"]) == h
    assert out["partition"] == "20 7 8"
    rows, cols, sc = O.find_candidates(vix, 20, 3)
    cand = out["candidates"].split()
    assert int(cand[0]) == len(rows)
    assert cand[1:] == [f"{r},{c},{s}" for r, c, s in zip(rows.tolist(), cols.tolist(), sc.tolist())]
    wins, words = O.viewsheds(z, 15, 10, 5, rows, cols)
    n, pc = map(int, out["viewsheds"].split())
    assert n == len(rows) and pc == int(O.popcounts(words).sum())
    o = O.site(rows, cols, wins, words, 160, 140, 0.9, max_selected=30)
    st = out["site"].split()
    assert st[0] == o["stop"] and int(st[1]) == len(o["index"])
    assert st[2:] == [f"{i}:{g}" for i, g in zip(o["index"].tolist(), o["gain"].tolist())]
    cov = out["coverage"].split()
    assert float(cov[0]) == float(cov[1]) == o["coverage"][-1]
    g0, g1 = map(int, out["gain"].split())
    assert g0 == int(O.popcounts(words[:1]).sum())
    assert g1 == O.marginal_gain(wins[0], words[0], o["cum"], 160, 140)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_cli_baseline_configs_match_python_path(tmp_path, name):
    """The CLI at BASELINE configs 1, 2, 3 and 5 writes the same result CSV as
    the Python path (Engine over the same C-ABI), whose picks the large-config
    tests check against the oracle (test_gpu_large.py)."""
    import paper_2006_16783_b200 as T
    from paper_2006_16783_b200.configs import CONFIGS, params_for, run, setup_terrain
    cfg = CONFIGS[name]
    args = ["--synth", "--nrows", cfg.nrows, "--ncols", cfg.ncols, "--seed", cfg.terrain_seed, "--roughness",
            cfg.roughness, "--zmin", cfg.zmin, "--zmax", cfg.zmax, "--roi", cfg.roi, "--tx-height", cfg.height,
            "--rx-height", cfg.height, "--coverage", cfg.target, "--max-selected", cfg.max_selected, "--no-images"]
    if cfg.random_observers:
        args += ["--observers-random", cfg.random_observers, "--observer-seed", cfg.observer_seed]
    else:
        args += ["--samples", cfg.samples, "--per-block", cfg.per_block, "--block-width", cfg.block,
                 "--vix-seed", cfg.vix_seed]
    if cfg.water_rows:
        args += ["--water-rows", cfg.water_rows]
    _run(args, tmp_path)
    rows = _csv(tmp_path)
    with T.Engine(0) as e:
        setup_terrain(e, cfg)
        res = run(e, cfg, params_for(cfg))
    assert [(int(r), int(c), int(g)) for _, r, c, g, _ in rows] == list(
        zip(res["row"].tolist(), res["col"].tolist(), res["gain"].tolist()))
    assert [float(x[4]) for x in rows] == res["coverage"].tolist()
