"""Command line: ``python -m paper_2511_14923_b200 <gen-mps|sample|evaluate> ...``.

Mirrors the reference CLI's ``sample`` subcommand (cli.py:116-160) and its JSON run
manifest (cli.py:45-74: config echo, SHA-256 of inputs, versions, wall time, peak RSS,
throughput); exceptions map to exit codes 2/3/4 (cli.py:351-357, errors.py:8-29).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import platform
import resource
import sys
import time

import numpy as np

from .errors import GbsError, ValidationError
from .formats import load_counts_file, load_mps, save_clicks_text, save_counts, save_mps
from .mps import MPS
from .sampler import MpsSamplerConfig, batch_sample, chain_log_probability

__version__ = "0.1.0"


def _sha256(path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def _manifest(command, config, inputs, outputs, t0, extra=None) -> dict:
    import torch

    man = {
        "command": command,
        "config": config,
        "inputs": {str(p): _sha256(p) for p in inputs},
        "outputs": [str(p) for p in outputs],
        "versions": {"paper_2511_14923_b200": __version__, "numpy": np.__version__, "torch": torch.__version__,
                     "python": platform.python_version()},
        "wall_time_s": time.perf_counter() - t0,
        "peak_rss_kb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss,
    }
    if extra:
        man.update(extra)
    return man


def _emit(man: dict) -> None:
    json.dump(man, sys.stdout, indent=1, sort_keys=True)
    sys.stdout.write("\n")


def cmd_gen_mps(args) -> int:
    t0 = time.perf_counter()
    mps = MPS.random(args.modes, args.chi, args.dim, seed=args.seed)
    save_mps(mps, args.out)
    cfg = {k: v for k, v in vars(args).items() if k != "func"}
    _emit(_manifest("gen-mps", cfg, [], [args.out], t0,
                    extra={"bond_dims": mps.bond_dims, "bytes": mps.nbytes}))
    return 0


def cmd_sample(args) -> int:
    t0 = time.perf_counter()
    mps = load_mps(args.mps, device="cuda" if args.device_sites else None)
    config = MpsSamplerConfig(N=args.samples, seed=args.seed, alpha_sigma=args.alpha_sigma,
                              batch_size=args.batch_size, device=args.device)
    batch = batch_sample(config, mps, start=args.start)  # indices start..start+N-1: runs resume by range
    # the rows' sample indices and the displacement law travel with the counts, so `evaluate`
    # scores each row under its own streams (failed samples are dropped from batch.counts)
    save_counts(args.out, batch.counts, mps.D, seed=args.seed, alpha_sigma=args.alpha_sigma, indices=batch.indices)
    outputs = [args.out]
    if args.clicks_out:
        save_clicks_text(args.clicks_out, batch.counts, seed=args.seed)
        outputs.append(args.clicks_out)
    cfg = {k: v for k, v in vars(args).items() if k != "func"}
    _emit(_manifest("sample", cfg, [args.mps], outputs, t0, extra={
        "M": mps.M, "D": mps.D, "chi": mps.chi,
        "n_generated": batch.N, "n_failed": batch.n_failed, "n_flagged": batch.n_flagged,
        "per_sample_s": batch.per_sample_mean,
        "throughput_per_s": (batch.N / batch.wall_time) if batch.wall_time > 0 else 0.0,
    }))
    return 0


def _sigma_arg(text):
    """--alpha-sigma value: a float >= 0, or "none" for no displacement stream."""
    if text.lower() == "none":
        return None
    v = float(text)
    if not (v >= 0.0 and np.isfinite(v)):
        raise argparse.ArgumentTypeError("alpha-sigma must be a finite number >= 0 or 'none'")
    return v


_UNSET = object()


def cmd_evaluate(args) -> int:
    """Log joint probability of each count row under the MPS (teacher-forced chain on the GPU).
    Row i is scored under the streams of its own sample index and the displacement law the counts
    were drawn with, both read from the counts file (v2); a v1 file carries neither, so then
    --alpha-sigma and --start must be given explicitly."""
    t0 = time.perf_counter()
    mps = load_mps(args.mps, device="cuda" if args.device_sites else None)
    f = load_counts_file(args.counts)
    counts, D, seed = f["counts"], f["D"], f["seed"]
    if D != mps.D or counts.shape[1] != mps.M:
        raise ValidationError(f"counts file (M={counts.shape[1]}, D={D}) does not match the MPS (M={mps.M}, D={mps.D})")
    if args.alpha_sigma is not _UNSET:
        sigma = args.alpha_sigma
        if f["alpha_sigma"] != "unknown" and sigma != f["alpha_sigma"]:
            raise ValidationError(f"--alpha-sigma {sigma} contradicts the counts file's {f['alpha_sigma']}")
    elif f["alpha_sigma"] == "unknown":
        raise ValidationError("the counts file does not record alpha_sigma (v1 file): pass --alpha-sigma "
                              "(a number, or 'none' for no displacement)")
    else:
        sigma = f["alpha_sigma"]
    if f["indices"] is not None:
        if args.start is not None:
            raise ValidationError("the counts file records each row's sample index; --start does not apply")
        idx = f["indices"]
    else:
        if args.start is None:
            raise ValidationError("the counts file does not record sample indices (v1 file): pass --start")
        idx = args.start + np.arange(counts.shape[0], dtype=np.int64)
    config = MpsSamplerConfig(N=counts.shape[0], seed=seed if args.seed is None else args.seed,
                              alpha_sigma=sigma, batch_size=args.batch_size, device=args.device)
    t1 = time.perf_counter()
    logp = np.empty(counts.shape[0])
    # rows with consecutive sample indices are evaluated as one run (one stream window each)
    breaks = np.nonzero(np.diff(idx) != 1)[0] + 1
    for lo, hi in zip(np.r_[0, breaks], np.r_[breaks, len(idx)]):
        if hi > lo:
            logp[lo:hi] = chain_log_probability(mps, counts[lo:hi], config, start=int(idx[lo]))
    dt = time.perf_counter() - t1
    np.save(args.out, logp)
    fin = np.isfinite(logp)
    cfg = {k: (None if v is _UNSET else v) for k, v in vars(args).items() if k != "func"}
    _emit(_manifest("evaluate", cfg, [args.mps, args.counts], [args.out], t0, extra={
        "M": mps.M, "D": mps.D, "chi": mps.chi, "n": int(counts.shape[0]), "seed_used": config.seed,
        "alpha_sigma_used": sigma, "counts_file_version": f["version"],
        "n_in_support": int(fin.sum()), "mean_logp": float(logp[fin].mean()) if fin.any() else None,
        "throughput_per_s": counts.shape[0] / dt if dt > 0 else 0.0,
    }))
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2511_14923_b200", description="B200 displaced-MPS sampler")
    sub = p.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gen-mps", help="write a random row-orthonormal MPS (.gmps)")
    g.add_argument("--modes", type=int, required=True)
    g.add_argument("--chi", type=int, required=True)
    g.add_argument("--dim", type=int, required=True, help="physical dimension D")
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out", required=True)
    g.set_defaults(func=cmd_gen_mps)
    s = sub.add_parser("sample", help="draw photon-count samples on the GPU")
    s.add_argument("--mps", required=True)
    s.add_argument("--samples", type=int, required=True)
    s.add_argument("--start", type=int, default=0,
                   help="first sample index (counter streams): a run resumes or shards by index range")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--alpha-sigma", type=float, default=None, help="alpha ~ CN(0, sigma^2) per sample and mode")
    s.add_argument("--batch-size", type=int, default=None)
    s.add_argument("--device", type=int, default=0)
    s.add_argument("--device-sites", action="store_true", help="load sites straight into device memory")
    s.add_argument("--out", required=True, help="counts file (.gmpc)")
    s.add_argument("--clicks-out", default=None, help="also write counts > 0 in the reference's text format")
    s.set_defaults(func=cmd_sample)
    e = sub.add_parser("evaluate", help="log joint probability of count rows under the MPS (teacher forcing, GPU)")
    e.add_argument("--mps", required=True)
    e.add_argument("--counts", required=True, help="counts file (.gmpc) from `sample`")
    e.add_argument("--seed", type=int, default=None, help="stream seed (default: the counts file's)")
    e.add_argument("--start", type=int, default=None,
                   help="sample index of the first row (v1 counts files only; v2 files record every row's index)")
    e.add_argument("--alpha-sigma", type=_sigma_arg, default=_UNSET,
                   help="displacement law (default: the counts file's; required for v1 files; 'none' = no displacement)")
    e.add_argument("--batch-size", type=int, default=None)
    e.add_argument("--device", type=int, default=0)
    e.add_argument("--device-sites", action="store_true")
    e.add_argument("--out", required=True, help="log probabilities (.npy)")
    e.set_defaults(func=cmd_evaluate)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except GbsError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.exit_code
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return ValidationError.exit_code
