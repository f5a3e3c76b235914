"""Regenerate profiles/*summary*.txt and profiles/ncu_traffic.json from the
committed ncu reports (run here, no GPU needed):
    python tests/probe/profile_summary.py"""
import collections, csv, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
PROF = os.path.join(ROOT, "profiles")
# (name, report, launch row in the report, description)
CAPS = [("L1_dK", "r1b_fc_and_L1dK.ncu-rep", 3,
         "wgrad_kernel, nq=3 column shifts as B descriptor offsets, KP=64, 3 loader groups (PDL build)"),
        ("FC_fwd", "r1b_fc_and_L1dK.ncu-rep", 0, "fc_fwd_kernel<5>: mma.sync m16n8k16, cp.async I ring, split-K 18"),
        ("FC_dI", "r1b_fc_and_L1dK.ncu-rep", 1, "fc_dgrad_kernel: mma.sync, one wave of 3 CTAs/SM"),
        ("FC_dK", "r1b_fc_and_L1dK.ncu-rep", 2, "fc_dk_kernel<5>: mma.sync, bulk-copy image ring, split-K 9"),
        ("L1_dK_prev", "r1_wgrad_L1_dK.ncu-rep", 0, "wgrad_kernel, earlier r1 build (before PDL)"),
        ("L3_dK", "r1_wgrad_L3_dK.ncu-rep", 0, "wgrad_kernel (capture predates descriptor-shift mode: nq=1)"),
        ("L1_fwd", "r1_conv_L1_fwd.ncu-rep", 0, "conv_mma_kernel fwd, G=8 CC=4, row-box staging")]
# Round 2: rows layout (D1-outer), tests/probe/prof_r2.sh (run_rows_layer.py <layer> <op> 3, -s 2 -c 1)
CAPS_R2 = [("L1_dI", "r2_L1_dI.ncu-rep", 0, "rows_conv_kernel dI (flipped-kernel conv of dO padded by 2), N=32 per tap"),
           ("L1_fwd", "r2_L1_fwd.ncu-rep", 0, "rows_conv_kernel fwd, virtual-grid shifted windows, N=32 per tap"),
           ("L1_dK", "r2_L1_dK.ncu-rep", 0, "rows_wgrad_kernel, row-walk slots (p) x atoms (q), MN-major I^T / dO"),
           ("L2_fwd", "r2_L2_fwd.ncu-rep", 0, "rows_conv_kernel fwd stride 2 (merged phase planes), N=64"),
           ("L3_dI", "r2_L3_dI.ncu-rep", 0, "rows_conv_kernel dI, chunk-staged source (cstage), N=64"),
           ("L4_dI", "r2_L4_dI.ncu-rep", 0, "rows_fc_kernel mode 1 (FC dI GEMM, N=256 tiles, direct bf16 stores)")]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


# Round 2, final build (tests/probe/prof_r2b.sh): every rows kernel of the stack
CAPS_R2B = [("L%d_%s" % (l, o), "r2b_L%d_%s.ncu-rep" % (l, o), 0, desc) for (l, o, desc) in [
    (1, "fwd", "rows_walk_kernel fwd s1: 3 row taps stacked in N=96, 3 TMA+MMA streams"),
    (1, "dI", "rows_walk_kernel dI s1"),
    (1, "dK", "rows_wgrad_kernel"),
    (2, "fwd", "rows_walk_kernel fwd s2 (phase planes), 2 streams"),
    (2, "dI", "rows_conv_kernel dI s2 (output phases)"),
    (2, "dK", "rows_wgrad_kernel s2"),
    (3, "fwd", "rows_conv_kernel fwd, N=128 per tap"),
    (3, "dI", "rows_walk_kernel dI, N=192, one stream"),
    (3, "dK", "rows_wgrad_kernel"),
    (4, "fwd", "rows_fc_kernel mode 0 (split-K GEMM)"),
    (4, "dI", "rows_fc_kernel mode 1 (N=256 tiles, coalesced stores)"),
    (4, "dK", "rows_fc_kernel mode 2")]]
# Round 2, final build after dynamic strips + PDL weight packs (tests/probe/prof_r2c.sh)
CAPS_R2C = [("L%d_%s" % (l, o), "r2c_L%d_%s.ncu-rep" % (l, o), 0, desc) for (l, o, desc) in [
    (1, "fwd", "rows_walk_kernel fwd s1: 3 row taps stacked in N=96, 3 streams, dynamic strips"),
    (1, "dI", "rows_walk_kernel dI s1"),
    (1, "dK", "rows_wgrad_kernel"),
    (2, "fwd", "rows_walk_kernel fwd s2 (phase planes)"),
    (2, "dI", "rows_conv_kernel dI s2 (output phases)"),
    (2, "dK", "rows_wgrad_kernel s2"),
    (3, "fwd", "rows_conv_kernel fwd, N=128 per tap"),
    (3, "dI", "rows_walk_kernel dI, N=192"),
    (3, "dK", "rows_wgrad_kernel"),
    (4, "fwd", "rows_fc_kernel mode 0 (split-K GEMM)"),
    (4, "dI", "rows_fc_kernel mode 1 (N=256 tiles, coalesced stores)"),
    (4, "dK", "rows_fc_kernel mode 2")]]


# Round 2, the training step's tensor-core primary kernels (tests/probe/prof_r2_train.sh)
CAPS_R2T = [("P_fwd", "r2_P_fwd.ncu-rep", 0, "primary_tc_fwd_kernel<5,5>: im2col tile -> 2 MMAs 128x128x16, staged 512-B stores"),
            ("P_dK", "r2_P_dK.ncu-rep", 0, "primary_tc_dk_kernel<5,5>: dO^T MN-major TMA boxes x im2col, 8 MMAs 128x64x16 per tile")]


def full_summaries(caps, rnd, traffic, tag=None, src=None):
    tag = tag or "r%d" % rnd
    src = src or (PROF if rnd == 1 else PROF)
    out = ["# Round %d ncu --set full captures (one launch each, --clock-control none, bf16, 1 B200)" % rnd,
           "# commands: " + ("tests/probe/run_layer.py / capture_ops.py" if rnd == 1 else "tests/probe/prof_%s.sh" % tag) +
           " under ncu --set full -k regex:<kernel>",
           "# (cache control on: cold L2; shares/stalls matter, not the absolute time; dram writes still dirty",
           "#  in the 126 MB L2 when the kernel ends are not counted, so writes can read below the algorithmic bytes)",
           ""]
    for name, f, row, desc in caps:
        path = os.path.join(PROF, f)
        if not os.path.exists(path):
            path = os.path.join(ROOT, "gpurun_out", f)
        if not os.path.exists(path):
            continue
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r = list(csv.reader(raw.splitlines()))
        h, u, v = r[0], r[1], r[2 + row]
        where = "profiles/" + f if path.startswith(PROF) else f + ", summary only (report not committed)"
        out.append("[%s]  (%s)  %s" % (name, where, desc))
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append("  %-80s %s %s" % (k, v[i], u[i]))
                d[k] = (float(v[i].replace(",", "")), u[i])
        tb = int(d["dram__bytes_read.sum"][0] * SCALE[d["dram__bytes_read.sum"][1]] +
                 d["dram__bytes_write.sum"][0] * SCALE[d["dram__bytes_write.sum"][1]])
        traffic[name if tag in ("r2c", "r2t") else tag + "_" + name] = tb
        out.append("  %-80s %d" % ("dram read+write bytes per launch", tb))
        out.append("")
    open(os.path.join(PROF, "%s_ncu_full_summary.txt" % tag), "w").write("\n".join(out) + "\n")


def launches(rnd, cmd, tag=None):
    tag = tag or "r%d" % rnd
    rows = [r for r in csv.reader(open(os.path.join(PROF, "%s_stack_launches.csv" % tag))) if len(r) > 5]
    h, data = rows[0], rows[1:]
    iK, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg, tot = collections.OrderedDict(), 0.0
    for r in data:
        val = float(r[iV].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[iU], 1)
        k = re.sub(r"\(.*", "", r[iK]).split("::")[-1]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += val
        tot += val
    out = ["# %s launch list: ncu --metrics gpu__time_duration.sum --clock-control none" % tag,
           "# command: python bench.py %s --no-cpu-baseline (eager warm-up steps, graph capture," % cmd,
           "#          graph replays, L2 flush fills); ncu times are cold-cache and serialised: compare SHARES",
           "launches %d, total %.1f us" % (len(data), tot / 1e3)]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("%-22s n=%4d total=%9.1f us share=%5.1f%% avg=%7.1f us" % (k, n, t / 1e3, 100 * t / tot, t / n / 1e3))
    open(os.path.join(PROF, "%s_stack_launches_summary.txt" % tag), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    traffic = {}
    full_summaries(CAPS, 1, traffic)
    full_summaries(CAPS_R2, 2, traffic, tag="r2a")
    full_summaries(CAPS_R2B, 2, traffic, tag="r2b")
    full_summaries(CAPS_R2C, 2, traffic, tag="r2c")
    full_summaries(CAPS_R2T, 2, traffic, tag="r2t")
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from the ncu --set full "
                        "captures in profiles/ (tests/probe/profile_summary.py); unprefixed keys: round-2 final build "
                        "(r2c captures of the kernels bench.py times); r2b_*: before dynamic strips / PDL packs; r2a_*: earlier round-2 rows kernels; r1_*: "
                        "round-1 natural-layout kernels")
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    launches(1, "--steps 3 --warmup 3")
    launches(2, "--steps 2 --warmup 1", tag="r2")
    launches(2, "--steps 2 --warmup 1 --no-parity", tag="r2b")
    launches(2, "--steps 2 --warmup 1 --no-parity", tag="r2c")
    launches(2, "--config pcapsnet_train --steps 2 --warmup 1 --no-parity", tag="r2t")
