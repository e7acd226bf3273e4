"""Carry wisdom over a space change that only ADDS knobs.

When a kernel's space gains a tunable (e.g. advec_u's ``ysplit``), its
fingerprint — and so its kernel key and wisdom file name — changes
(reference kerneldef.py:215-218, space.py:202-222).  Every old record is still
a valid point of the new space with the new knobs at their defaults (same
binary, same launch geometry), so its measurement carries over unchanged:
this rewrites ``<name>-<old fp>.wisdom`` as ``<name>-<new fp>.wisdom`` with
the defaults added to each config (keep-best merged into an existing new
file) and removes the old file.

    python tools/migrate_wisdom.py --kernel advec_u --precision fp32 [--wisdom wisdom]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def migrate(kernel: str, precision: str, wisdom_dir: Path) -> Path | None:
    from paper_2303_12374_b200.stencils.definitions import definition_for
    from paper_2303_12374_b200.wisdom import WisdomFile, WisdomRecord, load_or_create, merge_wisdom, wisdom_path

    d = definition_for(kernel, precision)
    key = d.kernel_key()
    name = key.rsplit("-", 1)[0]
    defaults = d.space.default_config()[0]
    new_path = wisdom_path(wisdom_dir, key)
    olds = [p for p in sorted(wisdom_dir.glob(f"{name}-*.wisdom")) if p != new_path]
    if not olds:
        return None
    files = [load_or_create(wisdom_dir, key)]
    for old in olds:
        wf = WisdomFile.load(old)
        moved = WisdomFile(kernel_key=key, objective_name=wf.objective_name)
        for r in wf.records:
            cfg = dict(r.config)
            for k, v in defaults.items():
                cfg.setdefault(k, v)
            if not d.space.is_valid(cfg):
                raise ValueError(f"{old.name}: record {r.problem} is not valid in the new space")
            moved.records.append(WisdomRecord(r.device, r.problem, cfg, r.objective_seconds, r.provenance))
        files.append(moved)
    merge_wisdom(files).save(new_path)
    for old in olds:
        old.unlink()
    return new_path


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--precision", action="append", default=None)
    ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
    a = ap.parse_args(argv)
    for p in a.precision or ["fp32", "fp64"]:
        out = migrate(a.kernel, p, Path(a.wisdom))
        print(f"{a.kernel} {p}: {out or 'nothing to migrate'}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
