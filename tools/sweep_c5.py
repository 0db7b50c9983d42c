"""BASELINE.json configs[4] on ONE GPU: population 256..16,384 x graph n 1e4..1e6 (BA attach 5, k = 0.05 n),
one bench.py line per point, summarised as a markdown table (generations/s, evals/s in the loop, pure
evaluation, CPU baseline).  `python tools/sweep_c5.py > profiles/r01c_sweep_c5.md` on the B200."""
import json, subprocess, sys
rows = []
for wl, n in (("n1e4", "1e4"), ("n1e5", "1e5"), ("c4", "1e6")):
    for pop in (256, 1024, 4096, 16384):
        cmd = [sys.executable, "bench.py", "--workload", wl, "--pop", str(pop), "--steps", "10", "--warmup", "3"]
        if pop != 4096:
            cmd.append("--no-cpu-baseline")
        out = subprocess.run(cmd, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            rows.append((n, pop, None, out.stderr[-300:]))
            continue
        rows.append((n, pop, d, ""))
print("`step` = one generation driven through the stepwise operator C-ABI (`bench.py`'s `value`, one host synchronisation per generation);"
      " `library loop` = the same generations inside `gapa_cuda_run` (no per-generation host work).\n")
print("| n | population | step (ms) | generations/s | evals/s (loop) | library loop generations/s | evals/s (evaluation alone) | e2e evals/s (host buffers) | CPU evals/s (threads) |")
print("|---|---|---|---|---|---|---|---|---|")
for n, pop, d, err in rows:
    if d is None:
        print(f"| {n} | {pop} | failed: {err!r} | | | | | | |")
        continue
    cpu = d.get("cpu_baseline")
    lib = d.get("library_loop")
    print(f"| {n} | {pop} | {d['ms_per_step']:.3f} | {d['generations_per_sec']:.0f} | {d['value']:.3g} | "
          + (f"{lib['generations_per_sec']:.0f}" if lib else "") + " | "
          f"{d['fitness_evals_per_sec_kernels_only']:.3g} | {d['e2e']['value']:.3g} | "
          + (f"{cpu['value']:.3g} ({cpu['cores']}, {cpu['kind']})" if cpu else "") + " |")
