"""Golden outputs of the REFERENCE command line (pkg/src/jhsvd/cli.py) and
test generator (testgen.py), for the CLI / file-format parity tests
(tests/test_cli.py).  Test infrastructure: imports the reference from a
writable copy of /root/reference/pkg (see make_golden.py) and writes
``cli/``: the JHSV / CSV files of ``testgen``, the ``strategy gen`` tables,
and the ``svd run`` / ``svd dist`` JSON reports and ``bench`` CSV with the
wall-time fields removed.

    python tests/golden/make_cli_golden.py
"""

from __future__ import annotations

import contextlib
import io
import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "cli"
sys.path.insert(0, str(HERE))
from make_golden import _import_reference  # noqa: E402


def run(cli, argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def strip_wall(text: str) -> str:
    rep = json.loads(text)
    rep.pop("wall_time_s", None)
    rep["config"]["input"] = "<input>"
    return json.dumps(rep, indent=2) + "\n"


def main():
    j = _import_reference()
    from jhsvd import cli

    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir()
    cases = {}
    for kind, n, expand in (("rrow", 16, 1), ("mm", 32, 0), ("rcol", 8, 2), ("bl", 12, 0)):
        rc, text = run(cli, ["strategy", "gen", "--kind", kind, "--n", str(n),
                             "--expand", str(expand)])
        name = f"strategy_{kind}_{n}_x{expand}.txt"
        (OUT / name).write_text(text)
        cases[name] = rc
    # testgen files (definite and indefinite)
    for typ, n, seed in ((3, 64, 5), (2, 48, 9)):
        stem = f"tg_t{typ}_n{n}_s{seed}"
        rc, _ = run(cli, ["testgen", "--type", str(typ), "--n", str(n), "--seed", str(seed),
                          "--out", str(OUT / f"{stem}.jhsv"),
                          "--lambda", str(OUT / f"{stem}.csv")])
        cases[stem] = rc
    inp = str(OUT / "tg_t3_n64_s5.jhsv")
    lam = str(OUT / "tg_t3_n64_s5.csv")
    rc, text = run(cli, ["svd", "run", "--input", inp, "--lambda", lam, "--width", "16",
                         "--accumulate-v"])
    (OUT / "svd_run_t3_n64_w16.json").write_text(strip_wall(text))
    rc, text = run(cli, ["svd", "run", "--input", str(OUT / "tg_t2_n48_s9.jhsv"), "--lambda",
                         str(OUT / "tg_t2_n48_s9.csv"), "--width", "8", "--variant", "bo",
                         "--strategy", "mm"])
    (OUT / "svd_run_t2_n48_w8_bo_mm.json").write_text(strip_wall(text))
    trace = OUT / "svd_dist_trace.csv"
    rc, text = run(cli, ["svd", "dist", "--input", inp, "--lambda", lam, "--width", "8",
                         "--workers", "2", "--accumulate-v", "--trace", str(trace)])
    (OUT / "svd_dist_t3_n64_w8_g2.json").write_text(strip_wall(text))
    rc, text = run(cli, ["bench", "--orders", "32,64", "--types", "1,3", "--variants", "fb,bo",
                         "--width", "16", "--seed", "7"])
    rows = [",".join(line.split(",")[:-1]) for line in text.strip().splitlines()]
    (OUT / "bench_o32-64_t1-3.csv").write_text("\n".join(rows) + "\n")
    (OUT / "exit_codes.json").write_text(json.dumps(cases, indent=1, sort_keys=True) + "\n")
    # the reference's worker mappings (distsim.optimize_mapping) for g = 2, 4
    from jhsvd.distsim import Topology, optimize_mapping
    from jhsvd.strategy import make_strategy

    maps = {}
    for g in (2, 4):
        m = optimize_mapping(make_strategy("rrow", 2 * g), Topology(g))
        maps[str(g)] = {"assignments": [[list(pq) for pq in st] for st in m.assignments],
                        "moves": [[list(mv) for mv in st] for st in m.moves],
                        "fast_exchanges": m.fast_exchanges}
    (OUT / "mappings.json").write_text(json.dumps(maps) + "\n")


if __name__ == "__main__":
    main()
