"""The reference's CLI (proj/tools/veil_cli.cpp, which uses only the C ABI)
compiled unmodified against libveil.so (tools/cli: a CLI11 stand-in for the
absent vendor/ tree) and, for comparison, against the reference itself."""
import json
import os
import subprocess

import numpy as np
import pytest

import bindings
from common import read_png_rgba
from paper_2405_13364_b200.abi import (
    RENDER_ALPHA_THRESHOLD,
    RENDER_FORCE_HIGH_PATH,
    RENDER_VISUALIZE_ERRORS,
    default_params,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "cli", "_build", "veil_cli")
CLI_REF = os.path.join(ROOT, "tools", "cli", "_build", "veil_cli_ref")
needs_cli = pytest.mark.skipif(not (os.path.exists(CLI) and os.path.exists(CLI_REF)),
                               reason="tools/cli not built (needs /root/reference at build time)")


def run(exe, *args):
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)


@needs_cli
def test_cli_links_libveil_and_parses():
    assert "libveil.so" in subprocess.run(["ldd", CLI], capture_output=True, text=True).stdout
    assert run(CLI, "--help").returncode == 0
    # CLI11 Range(1, 1024) on --depth-filter-size, exit code of a validation error
    assert run(CLI, "--scene", "synthetic:dense_bin", "--depth-filter-size", "2000").returncode != 0
    assert run(CLI, "--bogus").returncode != 0
    assert run(CLI).returncode == 1  # --scene or --compare is required


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--scene", "synthetic:dense_bin", "--seed", "3", "--width", "256", "--height", "256"],
    ["--scene", "synthetic:random_soup", "--seed", "5", "--width", "200", "--height", "150",
     "--depth-filter-size", "40", "--alpha-threshold"],
    ["--scene", "synthetic:intersecting_shells", "--seed", "2", "--width", "128", "--height", "96",
     "--force-high-path", "--visualize-errors", "--depth-filter-size", "1"],
])
def test_cli_on_libveil_equals_reference_cli(tmp_path, args):
    png = tmp_path / "ours.png"
    ours = run(CLI, *args, "--output", str(png), "--stats", str(tmp_path / "ours.json"))
    assert ours.returncode == 0, ours.stderr
    ref = run(CLI_REF, *args, "--stats", str(tmp_path / "ref.json"))
    assert ref.returncode == 0, ref.stderr
    a = json.loads((tmp_path / "ours.json").read_text())
    b = json.loads((tmp_path / "ref.json").read_text())
    for r in (a, b):
        r.pop("timings_us")
        r.pop("device", None)
    a["config"].pop("threads")
    b["config"].pop("threads")
    assert a == b
    # the PNG holds the reference's image
    kind = args[1].split(":")[1]
    seed, w, h = int(args[3]), int(args[5]), int(args[7])
    cfg = b["config"]
    flags = sum(f for k, f in (("alpha_threshold", RENDER_ALPHA_THRESHOLD),
                               ("visualize_errors", RENDER_VISUALIZE_ERRORS),
                               ("force_high_path", RENDER_FORCE_HIGH_PATH)) if cfg[k])
    img, _, _ = bindings.RefScene.synthetic(kind, seed, w, h).render(
        default_params(depth_filter_size=cfg["depth_filter_size"], flags=flags))
    assert np.array_equal(read_png_rgba(str(png)), img)
    diff = run(CLI, "--compare", str(png), str(png))
    assert diff.returncode == 0 and "0 differing pixels" in diff.stdout
