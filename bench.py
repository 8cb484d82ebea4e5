#!/usr/bin/env python
"""Forward+backward PD timestep throughput on B200 (BASELINE.json metric).

One step = one forward PD timestep (forward_step, reference forward.cpp:148-272)
plus its adjoint backward step (backward_step, backward.cpp:396-414) for the
canonical loss L = 1/2|q_T - rest|^2 + 1/2|v_T|^2 (drivers.cpp:384-396),
on the C3 workload: 103,680-tet heterogeneous (100x stiffness contrast)
Neo-Hookean crab-like block with Rayleigh damping folded into the factor.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (re-executed under torchrun when started plainly) runs the batched
system-ID configuration C5 — 64 parameter samples of the 30k-tet mesh sharded
over the ranks, one NCCL all-reduce of [loss, dL/dE] per evaluation — since a
single trajectory does not shard; --replicas keeps N
independent C3 trajectories instead.  Timing is the max over ranks.  The
reference arm times the CPU restatement of the reference (oracle/; the
reference itself cannot be built here: Eigen is absent) on the host cores,
the same warm-up and timed steps from the same start state.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
# the batch workload drives up to 32 sample streams concurrently; give each its
# own hardware work queue (must be set before the CUDA runtime starts)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, HERE)

PRODUCT_LIB = os.path.join(HERE, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so")
ORACLE_LIB = os.path.join(HERE, "oracle", "_build", "libheterodyn_oracle.so")
METRIC = "forward+backward PD timesteps/sec at 100k tets"
UNIT = "steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--workload", default="trajectory", choices=["trajectory", "batch"],
                    help="trajectory: one C3 trajectory per GPU (replicas for N>1); "
                         "batch: C5 batched system-ID, 64 C2 samples sharded over the GPUs + NCCL all-reduce")
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--frames", type=int, default=10, help="frames per sample trajectory (batch workload)")
    ap.add_argument("--ordering", default=None, help="factor ordering: nd-bfs (default), nd-geometric or metis")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=150.0,
                    help="seconds the CPU-baseline child may spend on its one fwd+bwd step (C4: ~2400)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent trajectories instead of the C5 batch shard")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def pin_device(local_rank: int, world: int):
    """One process per GPU: narrow visibility before any CUDA runtime starts, so
    the product library's runtime and torch's agree on the device."""
    if world <= 1:
        return
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    ids = [x for x in vis.split(",") if x.strip()] if vis else None
    os.environ["CUDA_VISIBLE_DEVICES"] = ids[local_rank] if ids else str(local_rank)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows = []
        self.proc = None

    def start(self):
        """Starts the poller and waits for its first row, so the timed region
        (as short as ~80 ms for C3) is sampled from its first millisecond."""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.i0 = len(self.rows)  # rows from here on fall in the timed region

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        n_in = len(self.rows) - self.i0
        t0 = time.time()  # a region shorter than the poll interval: the first row at its end
        while len(self.rows) - self.i0 < 1 and time.time() - t0 < 0.5:
            time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows[self.i0:self.i0 + max(n_in, 1)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


def measured_peak():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name="solve_traffic.json"):
    p = os.path.join(HERE, "profiles", name)
    try:
        with open(p) as f:
            return json.load(f).get("traffic_bytes_per_solve")
    except Exception:
        return None


def _oracle_step_worker(scene_json, q_path, v_path, out_path):
    import numpy as np
    from paper_2605_14526_b200.hd import Library
    lib = Library(ORACLE_LIB)
    sim = lib.scene(scene_json).sim()  # factorization: not timed
    sim.set_state(np.load(q_path), np.load(v_path), 0.0)
    sim.record(True)
    t0 = time.perf_counter()
    sim.step()
    sim.backward_canonical(download=False)
    dt = time.perf_counter() - t0
    with open(out_path, "w") as f:
        json.dump({"dt": dt, "iterations": sim.last_iterations, "contacts": sim.last_contact_count}, f)


def cpu_baseline(scene_dict, q, v, max_seconds=150.0):
    """Times the CPU restatement (oracle/, port of the reference) on one
    fwd+bwd step of the same workload from the same state, in a child process
    bounded by max_seconds (factorization excluded)."""
    import multiprocessing as mp
    import tempfile
    import numpy as np
    with tempfile.TemporaryDirectory() as d:
        qp, vp, op = os.path.join(d, "q.npy"), os.path.join(d, "v.npy"), os.path.join(d, "out.json")
        np.save(qp, q)
        np.save(vp, v)
        ctx = mp.get_context("spawn")
        p = ctx.Process(target=_oracle_step_worker, args=(json.dumps(scene_dict), qp, vp, op))
        t0 = time.perf_counter()
        p.start()
        p.join(max_seconds + 120.0)  # + factorization
        if p.is_alive():
            p.terminate()
            p.join()
            waited = time.perf_counter() - t0
            return {"value": 1.0 / waited, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                    "sample": f"1 fwd+bwd step did not finish within {waited:.0f} s (incl. factorization); "
                              f"value is an upper bound"}
        with open(op) as f:
            r = json.load(f)
    return {"value": 1.0 / r["dt"], "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"1 fwd+bwd step of the same workload from the GPU run's timed-region start state "
                      f"({r['dt']:.1f} s; forward iterations {r['iterations']}; contacts {r['contacts']}; "
                      f"factorization excluded)"}


WORKLOADS = {
    "C3": "100x E contrast, NH, alpha=0.05, beta0=0.01",
    "C4": "gripper pad: 100x E contrast NH (stiff core, soft pad), alpha=0.05, beta0=0.01, frictional contact "
          "(mu=0.5) against a rigid rounded cube edge",
    "C2": "NH nu=0.45, alpha=0.01",
    "C1": "corotated cantilever, x=0 face pinned",
}


def run_reference(args, scene_dict, world, rank):
    """Reference arm: the CPU restatement of the reference (oracle/) runs the
    GPU arm's schedule — W untimed warm-up steps from the scene's initial
    state, then K timed fwd+bwd steps (factorization excluded, as in the GPU
    arm) — on every host core of rank 0."""
    if rank != 0:
        return
    from paper_2605_14526_b200.hd import Library
    lib = Library(ORACLE_LIB)
    sc = lib.scene(scene_dict)
    t_fac = time.perf_counter()
    sim = sc.sim()
    t_fac = time.perf_counter() - t_fac
    warm = max(args.warmup, 3)
    for _ in range(warm):
        sim.record(True)
        sim.step()
        sim.backward_canonical(download=False)
        sim.record(False)
    times = []
    for _ in range(args.steps):
        sim.record(True)
        t0 = time.perf_counter()
        sim.step()
        sim.backward_canonical(download=False)
        times.append(time.perf_counter() - t0)
        sim.record(False)
    total = sum(times)
    val = len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": len(times),
        "warmup": warm, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the GPU arm's workload description, verbatim (same scene, same schedule)
        "config": {"workload": f"{args.config}: {scene_dict['name']} ({sc.element_count} tets, {sc.vertex_count} vertices, "
                               f"{WORKLOADS.get(args.config.upper(), '')})",
                   "parallelism": "replicas" if world > 1 else "single", "factorization_s": t_fac},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{warm} warm-up + {len(times)} timed fwd+bwd steps from the scene's initial "
                                   f"state (the GPU arm's schedule), CPU restatement of the reference (Eigen absent: "
                                   f"reference not buildable), HETERODYN_THREADS="
                                   f"{os.environ.get('HETERODYN_THREADS', 'all')}"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


BATCH_METRIC = "forward+backward PD timesteps/sec, batched system-ID (C5: 64 x 30k-tet samples)"


def batch_setup(args):
    from paper_2605_14526_b200 import scenes
    scene_dict = scenes.config_scene("C2", frames=args.frames)
    return scene_dict


def run_batch_reference(args, world, rank):
    """Reference arm of the batch workload: the CPU restatement evaluates a
    bounded sample of the batch (one sample's trajectory) on the host cores."""
    if rank != 0:
        return
    import numpy as np
    from paper_2605_14526_b200 import scenes
    from paper_2605_14526_b200.hd import Library
    lib = Library(ORACLE_LIB)
    scene_dict = batch_setup(args)
    sc = lib.scene(scene_dict)
    young = scenes.c5_young(args.samples, sc.element_count)
    frames = min(args.frames, 2)
    times = []
    t_all = time.perf_counter()
    for s in range(max(1, min(args.steps, 3))):
        b = sc.batch(1, young[s:s + 1])
        t0 = time.perf_counter()
        b.evaluate(frames)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > 120:
            break
    val = frames * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": BATCH_METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "warmup": 0, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5: {args.samples} samples of {scene_dict['name']}, {args.frames} frames each"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{len(times)} samples x {frames} frames fwd+bwd (factorization included per "
                                   f"sample, as the reference refactors per parameter sample)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_batch(args, world, rank):
    """C5: the batch's samples shard over the ranks (contiguous blocks); each
    rank evaluates its samples concurrently on one GPU and the [sum L, sum
    dL/dE] vectors are all-reduced over NCCL — the only cross-GPU traffic."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_14526_b200 import scenes
    from paper_2605_14526_b200.dist import allreduce_loss_grad, max_over_ranks, shard
    from paper_2605_14526_b200.hd import Library
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    lib = Library(PRODUCT_LIB)
    scene_dict = batch_setup(args)
    sc = lib.scene(scene_dict)
    ne, nv = sc.element_count, sc.vertex_count
    young = scenes.c5_young(args.samples, ne)
    mine = shard(args.samples, rank, world)
    # target: the trajectory end state at the nominal modulus (the "measurement")
    ref = sc.sim()
    ref.step(args.frames)
    target = ref.positions()
    del ref
    threads = max(1, min(len(mine), int(os.environ.get("HETERODYN_BATCH_THREADS", "32"))))
    t_build = time.perf_counter()
    b = sc.batch(len(mine), young[mine.start:mine.stop], threads=threads)
    t_build = time.perf_counter() - t_build
    b.set_target(target)
    buf = torch.zeros(1 + ne, dtype=torch.float64, device="cuda")
    def reduced():  # the all-reduce reads buf: finish it before the next evaluation writes buf
        allreduce_loss_grad(buf)
        torch.cuda.current_stream().synchronize()

    for _ in range(max(args.warmup, 3)):
        b.evaluate(args.frames, device_out=buf.data_ptr(), want_host=False)
        reduced()
    launches0 = b.kernel_launches
    solves0 = b.solve_count
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    dev_ms = 0.0
    for _ in range(args.steps):
        b.evaluate(args.frames, device_out=buf.data_ptr(), want_host=False)
        dev_ms += b.last_ms
        reduced()
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = b.kernel_launches - launches0
    solves = b.solve_count - solves0
    units = args.samples * args.frames * args.steps  # sample-timesteps, all ranks
    value = units / (ms / 1e3)
    total = buf.cpu().numpy()

    # e2e: target upload + evaluation + loss/gradient download through the C ABI
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_h = torch.from_numpy(np.ascontiguousarray(target)).pin_memory()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        b.set_target(t_h.numpy())
        r = b.evaluate(args.frames, device_out=buf.data_ptr(), want_host=True)
        reduced()
        host_total = buf.cpu()
    e3.record()
    e3.synchronize()
    ms_e2e = max_over_ranks(e2.elapsed_time(e3))
    e2e = units / (ms_e2e / 1e3)

    # one system-ID parameter update: every sample of this rank refactors
    t_ref = time.perf_counter()
    b.set_young(young[mine.start:mine.stop] * 1.0001)
    t_ref = time.perf_counter() - t_ref
    # L-BFGS-shaped steps: a parameter update (device refactorization of every
    # sample) before each evaluation — the throughput a system-ID loop sees
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e4 = torch.cuda.Event(enable_timing=True)
    e5 = torch.cuda.Event(enable_timing=True)
    e4.record()
    for k in range(args.steps):
        b.set_young(young[mine.start:mine.stop] * (1.0 + 1e-4 * (k + 2)))
        b.evaluate(args.frames, device_out=buf.data_ptr(), want_host=False)
        reduced()
    e5.record()
    e5.synchronize()
    ms_upd = max_over_ranks(e4.elapsed_time(e5))
    b.set_young(young[mine.start:mine.stop])

    # roofline of the dominant kernel: the batch's solve (lockstep: one
    # launch per pass streams every sample's block of the block-diagonal
    # factor), timed alone with CUDA events on the engine's stream; the
    # aggregate solve streaming over the whole step and the single-sample
    # solve are reported beside it
    ms_launch, bytes_launch = b.time_solve(20)
    probe = sc.sim()
    ms_solve, bytes_solve = probe.time_solve(50)
    peak, peak_kind = measured_peak()
    achieved = bytes_launch / (ms_launch / 1e3) / 1e9
    step_solve_gbs = solves * b.solve_bytes / (ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from paper_2605_14526_b200.hd import Library as L2
            o = L2(ORACLE_LIB).scene(scene_dict)
            ob = o.batch(1, young[:1])
            t0 = time.perf_counter()
            ob.evaluate(2)
            dt = time.perf_counter() - t0
            cpu = {"value": 2 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"1 sample x 2 frames fwd+bwd of the same batch ({dt:.1f} s, factorization included)"}
        except Exception as exc:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    if rank == 0:
        line = {
            "metric": BATCH_METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5: {args.samples} samples of {scene_dict['name']} ({ne} tets, {nv} vertices, "
                                   f"NH nu=0.45, beta0=0), E_s = 1e5 exp(0.5 z_s), mt19937_64 seed 2605, "
                                   f"{args.frames} frames fwd+bwd per sample per step",
                       "parallelism": f"samples sharded dp{world}, NCCL all-reduce of [loss, dL/dE] "
                                      f"({(1 + ne) * 8} B) per step",
                       "samples_per_rank": len(mine), "host_threads_per_rank": threads,
                       "batch_engine": "lockstep (one segmented engine per rank)" if b.lockstep else "one engine per sample",
                       "engine_build_s": t_build, "set_young_s": t_ref,
                       "steps_per_s_with_refactorization": units / (ms_upd / 1e3),
                       "l2_policy": "per-sample factors 64 x ~%.0f MB exceed L2" %
                                                               (probe.factor_nnz * 8 / 1e6),
                       "device_busy_ms_per_step": dev_ms / args.steps,
                       "loss_sum": float(total[0])},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 3 * nv * 8,
                    "d2h_bytes_per_step": (len(mine) + ne) * 8 + (1 + ne) * 8},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic("solve_traffic_c5.json"),
                         "traffic_scope": "DRAM bytes of one sample's solve (ncu capture, profiles/solve_traffic_c5.json)"
                                          " vs its algorithmic bytes",
                         "kernel": ("hdk_apply_inverse3 on the lockstep batch's block-diagonal factor (all of the rank's "
                                    "samples in one launch per pass)" if b.lockstep else
                                    "hdk_apply_inverse3 of one sample's factor"),
                         "bytes_per_launch": bytes_launch, "ms_per_launch": ms_launch,
                         "step_solve_streaming_gbs": step_solve_gbs,
                         "step_solve_streaming_frac": step_solve_gbs / peak,
                         "sample_solves_per_step": solves / args.steps,
                         "single_sample_solve_ms": ms_solve, "single_sample_solve_gbs": bytes_solve / (ms_solve / 1e3) / 1e9,
                         "peak_source": peak_kind},
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """--gpus N > 1 outside torchrun: re-exec this script as N ranks (one
    process per GPU) on 127.0.0.1, the way the driver launches it."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    world, rank, local = dist_env()
    if world > 1 and args.workload == "trajectory" and not args.replicas:
        # one trajectory does not shard: the multi-GPU
        # configuration is the batched system-ID C5 (samples sharded, NCCL
        # all-reduce of [loss, dL/dE]); --replicas keeps N C3 trajectories
        args.workload = "batch"
    pin_device(local, world)
    from paper_2605_14526_b200 import scenes
    if args.workload == "batch":
        if args.impl == "reference":
            if world > 1:
                import torch.distributed as dist
                dist.init_process_group("gloo", init_method="env://")
            run_batch_reference(args, world, rank)
            if world > 1:
                dist.barrier()
                dist.destroy_process_group()
            return
        if not os.path.exists(PRODUCT_LIB):
            raise SystemExit(f"product library missing: {PRODUCT_LIB} (run __graft_entry__.build())")
        run_batch(args, world, rank)
        return
    scene_dict = scenes.config_scene(args.config, ordering=args.ordering)
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo", init_method="env://")
        run_reference(args, scene_dict, world, rank)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import numpy as np
    import torch
    from paper_2605_14526_b200.hd import Library
    if not os.path.exists(PRODUCT_LIB):
        raise SystemExit(f"product library missing: {PRODUCT_LIB} (run __graft_entry__.build())")
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method="env://")
    lib = Library(PRODUCT_LIB)
    sc = lib.scene(scene_dict)
    t_fac = time.perf_counter()
    sim = sc.sim()
    t_fac = time.perf_counter() - t_fac
    n = sim.n
    ne = sc.element_count
    stream = torch.cuda.ExternalStream(sim.stream)

    contacts = []
    split = []  # (forward ms, backward ms) per timed step, CUDA events on the engine stream

    def one_step(timed=False):
        if timed:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(stream)
        sim.record(True)
        sim.step()
        it_f = sim.last_iterations
        contacts.append(sim.last_contact_count)
        if timed:
            ev[1].record(stream)
        sim.backward_canonical(download=False)
        sim.record(False)
        if timed:
            ev[2].record(stream)
            split.append(ev)
        return it_f

    for _ in range(max(args.warmup, 3)):
        one_step()
    q_start = sim.positions()
    v_start = sim.velocities()
    t_start = lib.lib.hd_sim_time(sim.h)

    # ---- device-resident throughput (value) ---------------------------------
    solves0 = sim.solve_count
    streams0 = sim.factor_streams
    launches0 = sim.kernel_launches
    fwd_its, bwd_its = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        fwd_its.append(one_step(timed=True))
        bwd_its.append(lib.lib.hd_sim_backward_iterations(sim.h))
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    fwd_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in split]))
    bwd_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in split]))
    launches = sim.kernel_launches - launches0
    solves = sim.solve_count - solves0
    streams = sim.factor_streams - streams0  # a multi-column solve of 8 contact columns streams the factor once
    from paper_2605_14526_b200.dist import max_over_ranks, replica_value
    ms = max_over_ranks(ms)
    if world > 1:
        dist.barrier()
    value = replica_value(args.steps, ms, world)

    # ---- end to end through the C ABI with host buffers (e2e) ----------------
    q_h = torch.from_numpy(q_start.copy()).pin_memory()
    v_h = torch.from_numpy(v_start.copy()).pin_memory()
    outs = {k: torch.zeros(n, dtype=torch.float64).pin_memory() for k in ("q", "v", "dq0", "dv0", "df")}
    de_h = torch.zeros(ne, dtype=torch.float64).pin_memory()
    import ctypes as C
    D = C.POINTER(C.c_double)
    ptr = lambda t: C.cast(t.data_ptr(), D)
    h2d = 2 * n * 8
    d2h = (5 * n + ne) * 8
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    t_h = t_start  # the e2e steps replay the timed region's steps (same states, same times)
    contacts_e2e = []
    for _ in range(args.steps):
        lib.check(lib.lib.hd_sim_set_state(sim.h, ptr(q_h), ptr(v_h), t_h))
        lib.check(lib.lib.hd_sim_record(sim.h, 1))
        lib.check(lib.lib.hd_sim_step(sim.h))
        t_h = lib.lib.hd_sim_time(sim.h)
        contacts_e2e.append(sim.last_contact_count)
        lib.check(lib.lib.hd_sim_backward_canonical(sim.h, ptr(outs["dq0"]), ptr(outs["dv0"]), ptr(outs["df"]),
                                                    ptr(de_h), None, 0))
        lib.check(lib.lib.hd_sim_positions(sim.h, ptr(outs["q"]), n))
        lib.check(lib.lib.hd_sim_velocities(sim.h, ptr(outs["v"]), n))
        lib.check(lib.lib.hd_sim_record(sim.h, 0))
        q_h.copy_(outs["q"])
        v_h.copy_(outs["v"])
    e3.record(stream)
    e3.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    ms_e2e = max_over_ranks(ms_e2e)
    e2e = replica_value(args.steps, ms_e2e, world)

    # ---- roofline of the dominant kernel (global solve) ---------------------
    ms_solve, bytes_solve = sim.time_solve(50)
    peak, peak_kind = measured_peak()
    achieved = bytes_solve / (ms_solve / 1e3) / 1e9
    nnz = sim.factor_nnz
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(), "kernel": "hdk_apply_inverse3 (S' row-dot + column-tile passes, 3 axes)",
                "bytes_per_launch": bytes_solve, "ms_per_launch": ms_solve, "peak_source": peak_kind}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(scene_dict, q_start, v_start, max_seconds=args.cpu_budget)
        except Exception as exc:  # reported, never fatal for the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        # factor streams timed as single solves (a multi-column stream costs more: a lower bound)
        step_share = ms_solve * streams / args.steps / (ms / args.steps)
        # whole-step algorithmic bytes (SURVEY.md §8(d) with this layout: S' read
        # twice per factor stream at 8 B per value, no indices; a multi-column
        # stream reads it once for all its columns): streams x 16 nnz(S') +
        # solves x 96 n (rhs / partials / z per column) + per adjoint iteration
        # a B apply (320 B/element) and the backbone's vectors — CG: 24 x 24 B
        # per vertex (A p with its CSR row, q, x / r, the z fold, p); Anderson:
        # 2 x (2m + 4) x 24 B, m = 8 — + per forward iteration a local sweep
        # (100 B/element) and its vectors (20 x 24 B per vertex) + the cache /
        # energy sweeps (3 x 100 B/element)
        n_fwd, n_bwd = float(np.mean(fwd_its)), float(np.mean(bwd_its))
        nv = sc.vertex_count
        factor_bytes = 16.0 * nnz
        vec_b = 960.0 if os.environ.get("HETERODYN_ADJOINT", "pcg") == "aa" else 576.0
        step_bytes = (streams / args.steps * factor_bytes + solves / args.steps * (bytes_solve - factor_bytes)
                      + n_bwd * (320.0 * ne + vec_b * nv) + n_fwd * (100.0 * ne + 480.0 * nv) + 300.0 * ne)
        step_gbs = step_bytes / (ms / args.steps / 1e3) / 1e9
        step_roofline = {"bytes_per_step": step_bytes, "achieved_gbs": step_gbs, "frac": step_gbs / peak,
                         "formula": "streams*16 nnz(S') + solves*96 n + N_bwd*(320 n_e + %d n_v) + N_fwd*(100 n_e + "
                                    "480 n_v) + 300 n_e" % vec_b}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {scene_dict['name']} ({ne} tets, {sc.vertex_count} vertices, "
                                   f"{WORKLOADS.get(args.config.upper(), '')})",
                       "parallelism": "replicas" if world > 1 else "single",
                       "factor": {"ordering": f"{args.ordering or 'nd-mvc'} (postordered)", "nnz_S": nnz, "free_vertices": sim.free_count,
                                  "build_s": t_fac},
                       "l2_policy": "inputs larger than L2 (factor values %.0f MB > 126 MB L2)" % (nnz * 8 / 1e6),
                       "mean_forward_iterations": float(np.mean(fwd_its)),
                       "mean_adjoint_iterations": float(np.mean(bwd_its)),
                       "forward_ms": fwd_ms, "backward_ms": bwd_ms,
                       "step_ms": [round(e[0].elapsed_time(e[2]), 3) for e in split],
                       "contacts_per_step": [int(x) for x in contacts[-args.steps:]],
                       "adjoint_iterations_per_step": [int(x) for x in bwd_its],
                       "solves_per_step": solves / args.steps,
                       "factor_streams_per_step": streams / args.steps,
                       "mean_contacts": float(np.mean(contacts[-args.steps:])),
                       "mean_contacts_e2e": float(np.mean(contacts_e2e)),
                       "solve_share_of_step_est": step_share,
                       "step_roofline": step_roofline},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
