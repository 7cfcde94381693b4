"""Command-line surface of the B200 engine (the reference's ``reduce`` and
``gen`` commands, cli.py:33-50,83-91, with the engine choice ``b200``).

Exit codes as the reference (cli.py:17-20): 0 ok, 1 infeasible, 2 input
error.  Instance files go through the native parser / serializer
(``mhsk_parse_instance``), so multi-GB instances never become Python tuples.

    python -m paper_2109_06042_b200 reduce -i inst.txt --rules dp,md --loop -o kernel.txt
    python -m paper_2109_06042_b200 gen --n 100000 --m 100000 --p 0.01 --alpha 3 -o c4.txt
"""

from __future__ import annotations

import argparse
import sys

from .instance import InstanceError, parse_instance_csr

EXIT_OK = 0
EXIT_INFEASIBLE = 1
EXIT_INPUT = 2


def _write_text(path: str, text: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)


def _cmd_reduce(args) -> int:
    from ._native import serialize_instance_text
    from .pipeline import PipelineSpec, run_pipeline

    with open(args.input, "r", encoding="utf-8") as fh:
        csr = parse_instance_csr(fh.read())
    phases = tuple(p.strip() for p in args.rules.split(",") if p.strip())
    spec = PipelineSpec(phases=phases, engine=args.engine, loop=args.loop, workers=args.workers)
    reduced, report = run_pipeline(csr, spec)
    if args.output:
        _write_text(args.output, serialize_instance_text(reduced))
    if args.report:
        _write_text(args.report, report.to_json() + "\n")
    else:
        print(report.to_json())
    return EXIT_INFEASIBLE if report.infeasible else EXIT_OK


def _cmd_gen(args) -> int:
    from ._native import serialize_instance_text
    from .generate import counter_random, generate_random

    if args.generator == "reference":
        csr = generate_random(args.n, args.m, args.p, args.alpha, args.seed).csr
    elif args.device:
        from ._native import context

        csr, _ = context().generate_random(args.n, args.m, args.p, args.alpha, args.seed)
    else:
        from ._native import generate_random_host

        csr = generate_random_host(args.n, args.m, args.p, args.alpha, args.seed)
    text = serialize_instance_text(csr)
    if args.output:
        _write_text(args.output, text)
    else:
        sys.stdout.write(text)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2109_06042_b200",
                                     description="B200 kernelization of Multiple Hitting Set instances.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("reduce", help="run a reduction pipeline on the GPU")
    p.add_argument("-i", "--input", required=True)
    p.add_argument("-o", "--output", help="write the reduced instance here")
    p.add_argument("--rules", default="dp,md", help="comma-separated phases from fe,dp,se,md")
    p.add_argument("--engine", choices=("b200",), default="b200")
    p.add_argument("--loop", action="store_true", help="repeat the phase list until nothing changes")
    p.add_argument("--report", help="write the JSON report here (default: stdout)")
    p.add_argument("--workers", type=int, default=1, help="accepted for compatibility (result-neutral)")
    p.set_defaults(func=_cmd_reduce)
    p = sub.add_parser("gen", help="generate a seeded random instance")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--p", type=float, required=True)
    p.add_argument("--alpha", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--generator", choices=("counter", "reference"), default="counter",
                   help="counter-based (host/device, bit-identical) or the reference's Mersenne-Twister draw")
    p.add_argument("--device", action="store_true", help="generate on the GPU (counter generator)")
    p.add_argument("-o", "--output")
    p.set_defaults(func=_cmd_gen)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (InstanceError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
