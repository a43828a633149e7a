#!/usr/bin/env python
"""Benchmark of the docking hot path (BASELINE.json configs[1]).

Workload (`cfg1-score-1M`): 1,000,000 random genotypes of one 40-atom /
8-torsion synthetic ligand (seeded), scored against 80^3
maps built on the GPU from a 4,000-atom synthetic receptor.  A step = one
fused pose+inter+intra pass over the 1M genotypes (per rank: weak scaling).

Arms
  default            our CUDA path.  `value`: genes resident in HBM, CUDA
                     events around each step's kernel, L2 flushed (256 MiB
                     write) before every timed step; `e2e`: the public
                     backend API with pinned host genes -> host results.
  --impl reference   the reference's CPU algorithm (the bit-exact C port in
                     oracle/, all host threads) on bounded samples of the
                     same workload; rank 0 only.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("OMP_WAIT_POLICY", "passive")  # oracle threads must not spin beside the GPU legs

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pose evaluations/sec"
UNIT = "poses/s"
N_POSES = 1_000_000
WORKLOAD = "cfg1-score-1M"
FP32_SPEC_TFLOPS = 2 * 128 * 148 * 1.965e9 / 1e12  # 74.4, spec-derived (no measured FP32 peak)
# dram__bytes_read.sum + dram__bytes_write.sum of one score_kernel launch (1M poses) from the
# committed ncu --set full capture; algorithmic HBM bytes = 120 MB genes + 20 MB results
TRAFFIC_BYTES = 166.14e6 + 20.66e6
TRAFFIC_SRC = "profiles/r2c_score.md (ncu --set full, one launch of score_kernel<0,64,4,1>)"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def build_inputs(device_grid: bool):
    from paper_2509_12232_b200 import chem, context, gridmaps, synth

    cfg = synth.CONFIGS[1]
    spec = synth.config_grid_spec(1)
    prot = synth.config_protein(1)
    lig = synth.config_ligand(1, 0)
    t0 = time.perf_counter()
    if device_grid:
        gset = gridmaps.build_grid_maps(prot, spec, cfg.probe_types)
        grid_src = "device (vd_grid_build)"
    else:
        from oracle import oracle

        w = chem.TermWeights()
        maps = oracle.build_grid(prot, spec.origin, spec.spacing, spec.dims, cfg.probe_types, w,
                                 chem.default_parameter_table(), n_threads=0)
        labels = list(cfg.probe_types) + [chem.ELEC_LABEL, chem.DESOLV_LABEL]
        gset = gridmaps.GridMapSet(spec, {l: maps[k] for k, l in enumerate(labels)})
        grid_src = "host (oracle C builder)"
    grid_s = time.perf_counter() - t0
    ctx = context.prepare_context(lig, gset)
    return gset, lig, ctx, grid_s, grid_src


def measured_peaks_file():
    """The driver-written MEASURED_PEAKS.json (HBM copy GB/s; no FP32 or L2 figure)."""
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def measure_peaks(grid_n=80, n_types=7):
    """Live hardware ceilings (tools/peaks.cu), best of 3 each:
    * fp32_ffma2_tflops: packed FFMA2 throughput (8 independent chains per thread);
    * l2_stream_gbs: coalesced L1-bypassing reads of a 32 MiB L2-resident buffer by every
      SM -- the L2 read bandwidth ceiling;
    * l2_sector_gbs: random whole 32-B sector reads of the same buffer -- the L2 ceiling
      for scattered sectors, the access grain of the trilinear gathers;
    * atom_pattern_gbs (context only): the score kernel's own 96-B atom pattern."""
    import ctypes

    path = ROOT / "tools" / "libvdpeaks.so"
    if not path.exists():
        return None
    lib = ctypes.CDLL(str(path))
    for f in ("vdp_fp32_peak_tflops", "vdp_l2_stream_gbs", "vdp_l2_sector_gbs",
              "vdp_atom_gather_gbs"):
        getattr(lib, f).restype = ctypes.c_double
    lib.vdp_l2_stream_gbs.argtypes = [ctypes.c_int64]
    lib.vdp_l2_sector_gbs.argtypes = [ctypes.c_int64]
    lib.vdp_atom_gather_gbs.argtypes = [ctypes.c_int, ctypes.c_int]
    return {"fp32_ffma2_tflops": max(lib.vdp_fp32_peak_tflops() for _ in range(3)),
            "l2_stream_gbs": max(lib.vdp_l2_stream_gbs(32 << 20) for _ in range(3)),
            "l2_sector_gbs": max(lib.vdp_l2_sector_gbs(32 << 20) for _ in range(3)),
            "atom_pattern_gbs": max(lib.vdp_atom_gather_gbs(grid_n, n_types) for _ in range(3))}


def roofline_block(t_launch, n_poses, fpp, ctx, inbox_frac, peaks, traffic=None,
                   traffic_src=None, kernel="vd::score_kernel<false,64,4,1>"):
    """SURVEY 8(d) rooflines of one kernel launch from hardware ceilings.

    Algorithmic work per pose is the reference's model (vd/bench.py:139-171):
    32 flops per pair + 107 per atom, and 96 gather bytes per atom -- counted here
    only for the in-box atoms, the only ones whose corners are loaded.  Ceilings:
    FP32 = the spec 2 x 128 lanes x 148 SMs x 1.965 GHz (the live FFMA2 probe beside
    it); L2 = the live coalesced L2-read probe (random-sector probe beside it); HBM =
    MEASURED_PEAKS.json.  The binding roof is the one with the lower poses/s ceiling."""
    n_atoms = int(ctx.n_atoms)
    per_s = n_poses / t_launch
    fp32_tf = fpp * per_s / 1e12
    fp32 = {"achieved": fp32_tf, "peak": FP32_SPEC_TFLOPS, "unit": "TFLOP/s",
            "frac": fp32_tf / FP32_SPEC_TFLOPS,
            "peak_source": "spec: 2 x 128 FP32 lanes x 148 SMs x 1.965 GHz",
            "flops_per_pose": fpp, "ceiling_poses_per_s": FP32_SPEC_TFLOPS * 1e12 / fpp}
    inbox_b = 96.0 * n_atoms * inbox_frac
    gather_gbs = inbox_b * per_s / 1e9
    gather = {"achieved": gather_gbs, "unit": "GB/s", "bytes_per_pose_inbox": inbox_b,
              "inbox_atom_fraction": inbox_frac,
              "model_bytes_per_pose_all_atoms": 96 * n_atoms,
              "achieved_model_all_atoms": 96.0 * n_atoms * per_s / 1e9}
    hbm_peak = measured_peaks_file().get("hbm_gbs")
    out = {"bound": "fp32", "achieved": fp32_tf, "peak": FP32_SPEC_TFLOPS, "unit": "TFLOP/s",
           "frac": fp32_tf / FP32_SPEC_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
           "kernel": kernel, "ms_per_launch": 1e3 * t_launch, "poses_per_launch": n_poses,
           "fp32": fp32, "l2_gather": gather}
    if peaks:
        fp32["measured_ffma2_tflops"] = peaks["fp32_ffma2_tflops"]
        fp32["frac_of_measured_ffma2"] = fp32_tf / peaks["fp32_ffma2_tflops"]
        l2 = peaks["l2_stream_gbs"]
        gather.update(peak=l2, frac=gather_gbs / l2,
                      peak_source="measured live: coalesced L1-bypassing LDG.128 reads of a 32 MiB "
                                  "L2-resident buffer by every SM (tools/peaks.cu), best of 3",
                      l2_sector_peak_gbs=peaks["l2_sector_gbs"],
                      frac_of_sector_peak=gather_gbs / peaks["l2_sector_gbs"],
                      atom_pattern_gbs_context=peaks["atom_pattern_gbs"],
                      ceiling_poses_per_s=l2 * 1e9 / inbox_b)
        out["arithmetic_intensity_flop_per_byte"] = fpp / inbox_b
        out["ridge_flop_per_byte"] = FP32_SPEC_TFLOPS * 1e3 / l2
        if gather["ceiling_poses_per_s"] < fp32["ceiling_poses_per_s"]:
            out.update(bound="l2-gather", achieved=gather_gbs, peak=l2, unit="GB/s",
                       frac=gather_gbs / l2)
    if traffic and hbm_peak:
        out["hbm"] = {"achieved": traffic / t_launch / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": traffic / t_launch / 1e9 / hbm_peak,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}
    return out


def flops_per_pose(ctx):
    # the reference's own model (vd/bench.py:139-171): 32 flops/pair + 107 flops/atom
    return 32 * ctx.n_pairs + 107 * ctx.n_atoms


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def smi_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v for v in vis.split(",") if v.strip()]
    if ids and all(v.strip().isdigit() for v in ids) and local_rank < len(ids):
        return int(ids[local_rank])
    return local_rank


def run_ours(args):
    import torch

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # any torchrun launch, even N=1
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2509_12232_b200 import _abi, synth
    from paper_2509_12232_b200.backend import CudaBackend

    _abi.ensure_device(local)
    gset, lig, ctx, grid_s, grid_src = build_inputs(device_grid=True)
    spec = gset.spec
    b = CudaBackend(mode="fast", device=local)
    grid, ligs = b.prepared(ctx)
    genes_h = synth.random_genes(rank, N_POSES, ctx.n_torsions, spec.origin, spec.upper)
    dev = torch.device("cuda", local)
    genes_d = torch.from_numpy(genes_h).to(dev)
    out_d = (torch.empty(N_POSES, dtype=torch.float64, device=dev),
             torch.empty(N_POSES, dtype=torch.float64, device=dev),
             torch.empty(N_POSES, dtype=torch.float32, device=dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def step():
        _abi.score_genes(grid, ligs, 0, genes_d, *out_d, mode=_abi.MODE_FAST, stream=sp)

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = _abi.launches()
    with ClockSampler(smi_index(local)) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        launches = _abi.launches() - l0
        if dist:
            dist.barrier()
        # keep the GPU busy a little longer so the sampler sees a loaded clock
        if clk.proc and len(clk.rows) < 3:
            t_end = time.time() + 0.5
            while time.time() < t_end:
                step()
            torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(z) for a, z in evs]
    t_loc = sum(ms) / 1e3
    t_max = t_loc
    if dist:
        tt = torch.tensor([t_loc], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = world * N_POSES * args.steps / t_max
    ms_per_step = 1e3 * t_max / args.steps

    # e2e: public API, pinned host genes in, host results out, copies inside the region
    pin_g = torch.from_numpy(genes_h).pin_memory()
    pin_out = (torch.empty(N_POSES, dtype=torch.float64).pin_memory(),
               torch.empty(N_POSES, dtype=torch.float64).pin_memory(),
               torch.empty(N_POSES, dtype=torch.float32).pin_memory())
    outs_np = tuple(t.numpy() for t in pin_out)
    g_np = pin_g.numpy()
    for _ in range(2):
        b.score_population_arrays(g_np, ctx, out=outs_np)
    e2e_steps = max(3, min(args.steps, 20))
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        b.score_population_arrays(g_np, ctx, out=outs_np)
    torch.cuda.synchronize(dev)
    te = time.perf_counter() - t0
    if dist:
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
    e2e_value = world * N_POSES * e2e_steps / te

    # sanity: device results agree with the oracle on a sample (not timed)
    from oracle import oracle

    from oracle import parity

    sub = slice(0, N_POSES, 61)  # 16,394 of the timed 1M poses
    we, wa, wt = oracle.dock_population(oracle.Ligand(ctx), genes_h[sub], n_threads=0)
    got = [o.cpu().numpy()[sub] for o in out_d]
    oks = [parity.within_tol(g, w) for g, w in zip(got, (we, wa, wt))]
    parity_ok = bool(all(o.all() for o in oks))
    parity_line = {"poses": int(len(wt)), "sample": "every 61st pose of the timed 1M batch",
                   "inter_within_tol": int(oks[0].sum()), "intra_within_tol": int(oks[1].sum()),
                   "total_within_tol": int(oks[2].sum()),
                   "max_rel_diff_total": float(np.max(np.abs(got[2].astype(np.float64) - wt)
                                                      / np.maximum(np.abs(wt), 1e-30))),
                   "tolerance": "|d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4 (north star)"}

    fpp = flops_per_pose(ctx)
    peaks = measure_peaks(int(spec.dims[0]), len(gset.maps) - 2)
    # share of atoms inside the grid box (the kernel gathers only for those; the reference's
    # model counts every atom), from the device pose path on a sample of the genes
    smp = b.pose_population(genes_h[:8192], ctx)
    lo_b, hi_b = np.asarray(ctx.box_lo, np.float32), np.asarray(ctx.box_hi, np.float32)
    inb = np.all((smp >= lo_b[None, :, None]) & (smp <= hi_b[None, :, None]), axis=1)
    inbox_frac = float(inb.mean())
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (pose stage f32/f64 bit-exact)",
        "data": "synthetic (SURVEY Appendix B recipes, seeded)",
        "config": {"workload": WORKLOAD, "poses_per_step_per_gpu": N_POSES,
                   "ligand_atoms": int(ctx.n_atoms), "torsions": int(ctx.n_torsions),
                   "pairs": int(ctx.n_pairs), "grid": "80^3 x 9 maps @0.375A",
                   "receptor_atoms": 4000, "mode": "fast",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": f"ligand/pose sharding x{world}, no data-path collective",
                   "grid_build_s": round(grid_s, 4), "grid_built_on": grid_src},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int(genes_h.nbytes),
                "d2h_bytes_per_step": int(N_POSES * (8 + 8 + 4)),
                "path": "CudaBackend.score_population_arrays (pinned numpy in/out)"},
        "roofline": roofline_block(t_loc / args.steps, N_POSES, fpp, ctx, inbox_frac, peaks,
                                   TRAFFIC_BYTES, TRAFFIC_SRC),
        "gpu_launches": int(launches),
        "parity_sample_ok": parity_ok,
        "parity": parity_line,
        "clocks": clk.summary(),
    }
    if args.screen_ligands > 0:
        line["screening"] = screening_leg(args, rank, world, dist, dev)
        if not args.csv:
            line["screening"].pop("_modeled", None)
        if args.csv and rank == 0:
            from paper_2509_12232_b200 import benchrecords as br

            s = line["screening"]
            fl, by = s.pop("_modeled")
            rec = br.make_record(s["workload"], "cuda", [s["ms"]], s["ligands"], fl, by,
                                 threads=world)
            br.emit_csv([rec], args.csv)
    if not args.no_extra:
        line["stress"] = stress_leg(args, rank, world, dist, dev)
        if rank == 0:
            line["single_dock"] = single_dock_leg(args, dev)
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(ctx, genes_h, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def screening_leg(args, rank, world, dist, dev):
    """cfg2-style virtual screen: ligands docked/s with the on-device GA (pop 256 x 200
    generations), ligands split by index over ranks, records all-gathered over NCCL."""
    import torch

    from paper_2509_12232_b200 import _abi, gridmaps, hostprep, synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.ga import GaConfig, _run
    from paper_2509_12232_b200.screening import gather_records, pack_records, shard_range

    cfg = synth.CONFIGS[2]
    spec = synth.config_grid_spec(2)
    gset = gridmaps.build_grid_maps(synth.config_protein(2), spec, cfg.probe_types)
    n = args.screen_ligands
    lo, hi = shard_range(n, rank, world)
    t0 = time.perf_counter()
    batch = hostprep.TopologyBatch.synth(2, lo, hi - lo)       # this rank's ligand range only
    arrays = hostprep.prepare_batch(batch, list(gset.maps))
    prep_s = time.perf_counter() - t0
    b = CudaBackend(mode="fast", device=dev.index)
    grid = b._grid_for_set(gset)
    lset = hostprep.ligand_set(arrays)
    gmax = 7 + int(batch.n_torsions.max())
    ga = GaConfig(population_size=256, generations=200,
                  translation_bounds=(spec.origin, spec.upper))
    count = hi - lo
    # warm-up: every ligand for two generations, so that each launch shape the batch uses has
    # been loaded (CUDA loads kernels lazily) and the stream-ordered allocator holds the buffers
    _run(grid, lset, 0, count, GaConfig(population_size=256, generations=2,
         translation_bounds=(spec.origin, spec.upper)), 0, lo, b._mode(), gmax, trace=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    bt, be, ba, bg, _, ne = _run(grid, lset, 0, count, ga, 0, lo, b._mode(), gmax,
                                 trace=False)
    ev1.record()
    torch.cuda.synchronize(dev)
    t_dock = ev0.elapsed_time(ev1) / 1e3
    t1 = time.perf_counter()
    rec = gather_records(pack_records(bt, be, ba, ne, bg, np.ones(len(bt))), n, dist)
    t_gather = time.perf_counter() - t1
    t_max = t_dock
    if dist:
        tt = torch.tensor([t_dock], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    evals = n * ga.population_size * (ga.generations + 1)
    # cuda-exact (the reference-equal numerics) on the same shard: its throughput prices
    # bit-exactness; its results are compared bit for bit with the oracle GA below
    _run(grid, lset, 0, count, GaConfig(population_size=256, generations=1,
         translation_bounds=(spec.origin, spec.upper)), 0, lo, _abi.MODE_EXACT, gmax, trace=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0.record()
    xbt, xbe, xba, xbg, _, _ = _run(grid, lset, 0, count, ga, 0, lo, _abi.MODE_EXACT, gmax,
                                    trace=False)
    ev1.record()
    torch.cuda.synchronize(dev)
    t_exact = ev0.elapsed_time(ev1) / 1e3
    if dist:
        tt = torch.tensor([t_exact], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_exact = float(tt.item())
    cpu, par = None, None
    if rank == 0:
        from oracle import oracle, parity

        stack = np.stack([gset.maps[l] for l in grid.labels]).astype(np.float32)
        ligs = oracle.ligands_from_arrays(arrays, stack, spec)
        par = {"tolerance": "|d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4 (north star)",
               "fast_best_rescored": parity.rescore_summary(ligs, bt, be, ba, bg),
               "exact_best_rescored": parity.rescore_summary(ligs, xbt, xbe, xba, xbg)}
        if not args.no_cpu:
            cpu, (k, og, obt) = cpu_screen_baseline(ligs, ga, spec, lo, args.cpu_seconds)
            params = oracle.ga_params(ga, spec.origin, spec.upper)
            ag = parity.ga_agreement(ligs[:k], params, 0, lo, bt[:k], bg[:k],
                                     oracle_out=(og, obt))
            rms = ag.pop("_rmsd")
            ag.pop("_oracle_best_total")
            ag["rmsd_of_disagreeing"] = [round(float(x), 3) for x in rms[~np.isnan(rms)]
                                         if x > 0.5]
            par["fast_vs_oracle_ga"] = ag
            par["exact_vs_oracle_ga"] = {
                "ligands": k, "bit_identical_best_total": int(np.sum(xbt[:k] == obt)),
                "bit_identical_best_genes": int(np.sum(np.all(xbg[:k, :og.shape[1]] == og, axis=1)))}
    from paper_2509_12232_b200 import benchrecords as br

    npairs = float(arrays["pair_start"][-1]) / max(1, count)
    modeled = br.modeled_work(npairs * n, float(batch.n_atoms.mean()) * n, ga.population_size,
                              ga.generations)
    return {"metric": "ligands docked/sec", "value": n / t_max, "unit": "ligands/s",
            "pose_evals_per_s": evals / t_max, "ligands": n, "ms": 1e3 * t_max,
            "ga": "pop 256 x 200 generations (cfg2 distribution, 64^3 grid, 3000-atom receptor)",
            "mode": "fast",
            "workload": ("cfg2-screen-10k" if n == 10000 else "cfg3-screen-100k" if n == 100000
                         else f"cfg2-distribution x{n}"),
            "gathered_records": int(rec.shape[0]), "gather_ms": round(1e3 * t_gather, 3),
            "host_prep_s_per_rank": round(prep_s, 3),
            "timing": "CUDA events around vd_dock_batch (generation-synchronous GA: per generation one pop_score_kernel and one ga_step_kernel launch per launch-shape group of ligands, groups concurrent on streams; the exact leg: one persistent GA launch per atom-count bucket), max over ranks",
            "exact_mode": {"value": n / t_exact, "unit": "ligands/s", "ms": 1e3 * t_exact,
                           "note": "the same batch with reference-exact scoring (fp64 sums in "
                                   "the reference's lane-8 order, libm-equal exp): bit-identical "
                                   "to the oracle GA"},
            **({"parity": par} if par else {}),
            **({"cpu_baseline": cpu} if cpu else {}),
            "_modeled": modeled}


def stress_leg(args, rank, world, dist, dev):
    """cfg4 (BASELINE configs[4]): 2,000 ligands of 128 atoms / 32 torsions, 126^3 x 10 maps
    from an 8,000-atom receptor (built on the device), GA pop 512 x 300 generations, ligands
    split by index over ranks; ligands/s device-timed, max over ranks."""
    import torch

    from paper_2509_12232_b200 import gridmaps, hostprep, synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.ga import GaConfig, _run
    from paper_2509_12232_b200.screening import shard_range

    spec = synth.config_grid_spec(4)
    t0 = time.perf_counter()
    gset = gridmaps.build_grid_maps(synth.config_protein(4), spec, synth.CONFIGS[4].probe_types)
    grid_s = time.perf_counter() - t0
    n = args.stress_ligands
    lo, hi = shard_range(n, rank, world)
    batch = hostprep.TopologyBatch.synth(4, lo, hi - lo)
    arrays = hostprep.prepare_batch(batch, list(gset.maps))
    b = CudaBackend(mode="fast", device=dev.index)
    grid = b._grid_for_set(gset)
    lset = hostprep.ligand_set(arrays)
    gmax = 7 + int(batch.n_torsions.max())
    bounds = (spec.origin, spec.upper)
    ga = GaConfig(population_size=512, generations=300, translation_bounds=bounds)
    _run(grid, lset, 0, min(4, hi - lo), GaConfig(population_size=512, generations=1,
         translation_bounds=bounds), 0, lo, b._mode(), gmax, trace=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    res = _run(grid, lset, 0, hi - lo, ga, 0, lo, b._mode(), gmax, trace=False)
    ev1.record()
    torch.cuda.synchronize(dev)
    t = ev0.elapsed_time(ev1) / 1e3
    if dist:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    # parity (outside the timed region): every rank-0 best re-scored by the oracle; the
    # oracle GA (also the CPU baseline) on the first ligands, compared with the device's
    bt, be, ba, bg, _, _ = res
    par, cpu = None, None
    if rank == 0:
        from oracle import oracle, parity

        stack = np.stack([gset.maps[l] for l in grid.labels]).astype(np.float32)
        ligs = oracle.ligands_from_arrays(arrays, stack, spec)
        par = {"tolerance": "|d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4 (north star)",
               "fast_best_rescored": parity.rescore_summary(ligs, bt, be, ba, bg)}
        if not args.no_cpu:
            cpu, (k, og, obt) = cpu_screen_baseline(ligs, ga, spec, lo, args.cpu_seconds,
                                                    label="cfg4")
            ag = parity.ga_agreement(ligs[:k], oracle.ga_params(ga, spec.origin, spec.upper), 0,
                                     lo, bt[:k], bg[:k], oracle_out=(og, obt))
            rms = ag.pop("_rmsd")
            ag.pop("_oracle_best_total")
            ag["rmsd_of_disagreeing"] = [round(float(x), 3) for x in rms[~np.isnan(rms)]
                                         if x > 0.5]
            par["fast_vs_oracle_ga"] = ag
    npairs = float(arrays["pair_start"][-1]) / max(1, hi - lo)
    return {"metric": "ligands docked/sec", "value": n / t, "unit": "ligands/s",
            **({"parity": par} if par else {}), **({"cpu_baseline": cpu} if cpu else {}),
            "pose_evals_per_s": n * 512 * 301 / t, "ligands": n, "ms": 1e3 * t,
            "workload": "cfg4-stress" if n == 2000 else f"cfg4-distribution x{n}",
            "ligand": f"{int(batch.n_atoms.max())} atoms, {int(batch.n_torsions.max())} torsions, "
                      f"{npairs:.0f} pairs on average",
            "ga": "pop 512 x 300 generations", "grid": "126^3 x 10 maps, 8000-atom receptor",
            "grid_build_s": round(grid_s, 3),
            "timing": "CUDA events around vd_dock_batch, max over ranks"}


def single_dock_leg(args, dev):
    """cfg0 (BASELINE configs[0]): one 32-atom / 6-torsion ligand, 48^3 maps from a 2,000-atom
    receptor, GA pop 100 x 50, seed 0, through the public ga.dock (context preparation
    included), 10 runs dropping the 3 slowest (vd/bench.py:97-98); the restated GA on one host
    core beside it."""
    import torch

    from oracle import oracle
    from paper_2509_12232_b200 import gridmaps, synth
    from paper_2509_12232_b200.backend import CudaBackend
    from paper_2509_12232_b200.context import prepare_context
    from paper_2509_12232_b200.ga import GaConfig, dock

    spec = synth.config_grid_spec(0)
    gset = gridmaps.build_grid_maps(synth.config_protein(0), spec, synth.CONFIGS[0].probe_types)
    topo = synth.config_ligand(0, 0)
    cfg = GaConfig(population_size=100, generations=50, seed=0)
    b = CudaBackend(mode="fast", device=dev.index)
    dock(topo, gset, cfg, backend=b)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        r = dock(topo, gset, cfg, backend=b)
        ts.append(time.perf_counter() - t0)
    gpu_s = float(np.mean(sorted(ts)[:7]))
    out = {"metric": "seconds per dock", "value": gpu_s, "unit": "s", "higher_is_better": False,
           "workload": "cfg0-single-dock", "best_total": float(r.best_score.total),
           "timing": "wall clock around ga.dock (host context prep + one GA launch + copies), "
                     "mean of the 7 fastest of 10"}
    from oracle import parity

    lig = oracle.Ligand(prepare_context(topo, gset))
    params = oracle.ga_params(cfg, spec.origin, spec.upper)
    og, obt, *_ = oracle.dock(lig, params, 0, 0)
    rx = dock(topo, gset, cfg, backend=CudaBackend(mode="exact", device=dev.index))
    out["parity"] = {
        "oracle_best_total": float(obt),
        "fast_within_tol": bool(parity.within_tol([r.best_score.total], [obt])[0]),
        "fast_best_pose_rmsd": parity.rmsd(lig, r.best_genotype, og),
        "exact_bit_identical": bool(np.float32(rx.best_score.total) == obt
                                    and np.array_equal(rx.best_genotype, og)),
        "tolerance": "|d| <= 1e-3 kcal/mol or |d|/|E| <= 1e-4, else RMSD <= 0.5 A"}
    if not args.no_cpu:
        cs = []
        for _ in range(10):
            t0 = time.perf_counter()
            oracle.dock(lig, params, 0, 0)
            cs.append(time.perf_counter() - t0)
        out["cpu_baseline"] = {"value": float(np.mean(sorted(cs)[:7])), "unit": "s", "cores": 1,
                               "kind": "port", "cpu_model": cpu_model(), "sample": "the same dock (restated GA, "
                               "oracle/vd_ga_oracle.c) on one host core, 7 fastest of 10"}
    return out


def cpu_screen_baseline(ligs, ga, spec, index_base, seconds=10.0, label="cfg2"):
    """The reference GA + scoring on the host (oracle/vd_ga_oracle.c: the restated GA with
    the device's per-ligand keys, oracle/vd_oracle.c scoring, OpenMP over ligands) on the
    first ligands of the batch, bounded to ~`seconds`: ligands docked/s on all host
    threads.  Also returns (k, best genes, best totals) of every ligand it docked (0..k-1),
    for the GA parity comparison."""
    from oracle import oracle

    cores = oracle.cores()
    params = oracle.ga_params(ga, spec.origin, spec.upper)
    k = min(len(ligs), cores)  # probe: one ligand per thread
    t0 = time.perf_counter()
    g0, b0, *_ = oracle.dock_many(ligs[:k], params, 0, index_base, n_threads=cores)
    t_probe = time.perf_counter() - t0
    rate = k / max(t_probe, 1e-9)
    m = int(min(len(ligs) - k, max(cores, rate * seconds)))
    if m <= 0 or rate * seconds < 2 * k:  # the probe already took the budget: report it
        value, first, n_s, dt, genes, bests = rate, 0, k, t_probe, g0, b0
    else:
        t0 = time.perf_counter()
        g1, b1, *_ = oracle.dock_many(ligs[k:k + m], params, 0, index_base + k, n_threads=cores)
        dt = time.perf_counter() - t0
        value, first, n_s = m / dt, k, m
        w = max(g0.shape[1], g1.shape[1])
        genes = np.zeros((k + m, w))
        genes[:k, :g0.shape[1]], genes[k:, :g1.shape[1]] = g0, g1
        bests = np.concatenate([b0, b1])
    cpu = {"value": value, "unit": "ligands/s", "cores": cores, "kind": "port",
           "cpu_model": cpu_model(),
           "sample": f"ligands {first}..{first + n_s - 1} of the {label} batch, pop "
                     f"{ga.population_size} x {ga.generations} generations, {dt:.1f} s on {cores} "
                     "threads (oracle/vd_ga_oracle.c restated GA + oracle/vd_oracle.c scoring)"}
    return cpu, (len(bests), genes, bests)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(ctx, genes, seconds=10.0):
    """The reference algorithm (bit-exact C port, all host threads) on the cfg1 genes:
    whole passes over the 1M genotypes (or a prefix) until ~`seconds` of CPU work."""
    from oracle import oracle

    lig = oracle.Ligand(ctx)
    cores = oracle.cores()
    n = min(len(genes), 16384)
    t0 = time.perf_counter()
    oracle.dock_population(lig, genes[:n], n_threads=cores)
    rate = n / max(time.perf_counter() - t0, 1e-9)
    n = int(min(len(genes), max(16384, rate * seconds)))
    reps = max(1, int(rate * seconds // n))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.dock_population(lig, genes[:n], n_threads=cores)
    dt = time.perf_counter() - t0
    return {"value": reps * n / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{reps} pass(es) over the first {n} of the {N_POSES} cfg1 genotypes, "
                      f"{dt:.1f} s on {cores} threads (oracle/vd_oracle.c, bit-exact restatement "
                      "of SimdBackend.dock_population)"}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    from oracle import oracle
    from paper_2509_12232_b200 import synth

    gset, lig, ctx, grid_s, grid_src = build_inputs(device_grid=False)
    spec = gset.spec
    per_step = args.ref_sample
    genes = synth.random_genes(0, per_step * 4, ctx.n_torsions, spec.origin, spec.upper)
    L = oracle.Ligand(ctx)
    cores = oracle.cores()
    for k in range(args.warmup):
        oracle.dock_population(L, genes[(k % 4) * per_step:((k % 4) + 1) * per_step], n_threads=cores)
    t0 = time.perf_counter()
    for k in range(args.steps):
        oracle.dock_population(L, genes[(k % 4) * per_step:((k % 4) + 1) * per_step], n_threads=cores)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "host_cores_only": True,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (SURVEY Appendix B recipes, seeded)",
        "config": {"workload": WORKLOAD, "poses_per_step": per_step, "grid_build_s": round(grid_s, 2),
                   "grid_built_on": grid_src},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} cfg1 genotypes per step (of the 1M workload); "
                                   "oracle/vd_oracle.c is bit-exact with the reference's simd "
                                   "backend (tests/test_oracle_golden.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():  # noqa: C901
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=16384)
    ap.add_argument("--csv", default=None, help="also write a BenchRecord CSV row (vd/bench.py schema)")
    ap.add_argument("--screen-ligands", type=int, default=None,
                    help="ligands for the screening leg (0 disables; default: cfg2's 10,000 at "
                         "--gpus 1, cfg3's 100,000 sharded at --gpus > 1)")
    ap.add_argument("--stress-ligands", type=int, default=2000,
                    help="cfg4 ligands for the stress leg")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the cfg4 stress and cfg0 single-dock legs")
    ap.add_argument("--launch-check", action="store_true",
                    help="CPU test of the rank launcher: gloo ranks, no GPU work")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.screen_ligands is None:  # BASELINE cfg2 (10k) on one GPU, cfg3 (100k) sharded
        args.screen_ligands = 10000 if args.gpus == 1 else 100000
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus)  # does not return
    world = env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.launch_check:
        launch_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def relaunch(n: int):
    """`python bench.py --gpus N` without torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1, exactly as the driver launches them."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def launch_check(args):
    """The launcher's contract without a GPU: every rank joins one gloo group of
    --gpus ranks, agrees on the max of a per-rank time, rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "launch_check": True, "n_gpus": world,
                          "max_over_ranks": float(t.item()),
                          "screen_ligands": args.screen_ligands}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
