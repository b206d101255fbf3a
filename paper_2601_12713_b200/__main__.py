"""Columnar command line (mirrors `dmlens analyze` / `dmlens audit`, cli.py:41-93, 126-236):

  python -m paper_2601_12713_b200 analyze TRACE [--json] [--min-bytes N] [--strict-pseudocode] [-q] [-v]
  python -m paper_2601_12713_b200 audit TRACE --payload-dir DIR [-q] [-v]
  python -m paper_2601_12713_b200 version

`analyze --oracle` (the reference's brute-force cross-check, cli.py:57-58,145-152) is
rejected with an explicit message: the brute-force oracles are test infrastructure here.

NDJSON is parsed natively (ingest.py), analysed on the GPU, filtered / summed /
rendered from columns (reporting.py) -- no per-event Python objects.  Exit codes
as the reference: 0 ok, 1 input error, 2 internal error.
"""
from __future__ import annotations

import argparse
import os
import sys

EXIT_OK, EXIT_INPUT, EXIT_INTERNAL = 0, 1, 2
WARN_REASON = "delete without a live allocation at this device address"


def _parser():
    ap = argparse.ArgumentParser(prog="b200lens")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("analyze")
    a.add_argument("trace")
    a.add_argument("--json", action="store_true")
    a.add_argument("--min-bytes", type=int, default=1)  # cli.py:61-63 (1 keeps everything)
    a.add_argument("--oracle", action="store_true")
    a.add_argument("--strict-pseudocode", action="store_true")
    a.add_argument("-q", "--quiet", action="store_true")
    a.add_argument("-v", "--verbose", action="store_true")
    u = sub.add_parser("audit")
    u.add_argument("trace")
    u.add_argument("payload_dir_pos", nargs="?", default=None, help=argparse.SUPPRESS)  # r01 positional form
    u.add_argument("--payload-dir", dest="payload_dir", default=None)  # cli.py:84-87
    u.add_argument("-q", "--quiet", action="store_true")
    u.add_argument("-v", "--verbose", action="store_true")
    sub.add_parser("version")
    return ap


def _color() -> bool:
    mode = os.environ.get("DMLENS_COLOR", "auto")
    return mode == "always" or (mode != "never" and sys.stdout.isatty())


def _load(path, validate=True):
    from .ingest import TraceIOError, parse_trace_columns
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError as exc:
        print(f"dmlens: error: cannot read {path}: {exc}", file=sys.stderr)
        return None
    try:
        return parse_trace_columns(data, validate=validate)
    except TraceIOError as exc:
        print(f"dmlens: error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return None


def cmd_analyze(args) -> int:
    if args.oracle:
        print("dmlens: error: --oracle is not supported by the B200 engine CLI (run `dmlens analyze --oracle`)",
              file=sys.stderr)
        return EXIT_INTERNAL
    from .analysis import analyze_columns
    from .reporting import build_report, filter_min_bytes, render_json, render_text
    from .analysis import EngineInvalid
    from .ingest import event_violations, invariant_error
    cols = _load(args.trace, validate=False)  # the analysis run below validates the events
    if cols is None:
        return EXIT_INPUT
    try:
        cf = analyze_columns(cols, strict=args.strict_pseudocode, with_savings=args.min_bytes <= 1)
    except EngineInvalid as exc:  # the same error parse_trace would have raised
        err = invariant_error(event_violations(cols, exc))
        print(f"dmlens: error: {type(err).__name__}: {err}", file=sys.stderr)
        return EXIT_INPUT
    if not args.quiet:
        for i in cf.warn_index.tolist():
            print(f"dmlens: warning: seq {int(cols.seq[i])}: {WARN_REASON}", file=sys.stderr)
    rep = build_report(cols, filter_min_bytes(cols, cf, args.min_bytes))
    if not args.quiet:
        for w in rep.warnings:
            print(f"dmlens: warning: {w}", file=sys.stderr)
    sys.stdout.write(render_json(rep) if args.json else render_text(rep, color=_color()))
    if args.verbose:
        print(f"dmlens: {cols.n} events, {sum(rep.counts.values())} findings", file=sys.stderr)
    return EXIT_OK


def cmd_audit(args) -> int:
    from pathlib import Path
    args.payload_dir = args.payload_dir or args.payload_dir_pos
    if args.payload_dir is None:
        print("dmlens audit: error: the following arguments are required: --payload-dir", file=sys.stderr)
        return EXIT_INTERNAL

    from .hashing import audit_payloads
    cols = _load(args.trace)
    if cols is None:
        return EXIT_INPUT
    hashes, payloads, missing = [], [], 0
    for i in range(cols.n):
        if int(cols.kind[i]) != 0 or int(cols.hash[i]) == 0 or int(cols.bytes[i]) == 0:
            continue
        seq = int(cols.seq[i])
        try:
            payloads.append((Path(args.payload_dir) / f"{seq}.bin").read_bytes())
        except OSError:
            missing += 1
            if not args.quiet:
                print(f"dmlens: warning: no payload sidecar for seq {seq}", file=sys.stderr)
            continue
        hashes.append(int(cols.hash[i]))
    collisions, _ = audit_payloads(hashes, payloads)
    if args.verbose:
        print(f"dmlens: audited {len(hashes)} transfers ({missing} missing sidecars)", file=sys.stderr)
    print(f"collision_count: {collisions}")
    return EXIT_OK


def cmd_version(args) -> int:
    from . import __version__
    print(f"dmlens {__version__}")
    return EXIT_OK


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return {"analyze": cmd_analyze, "audit": cmd_audit, "version": cmd_version}[args.cmd](args)
    except Exception as exc:  # noqa: BLE001 - the reference maps every internal failure to exit 2
        print(f"dmlens: internal error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
