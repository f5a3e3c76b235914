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


def full_summaries():
    out = ["# Round 1 ncu --set full captures (one launch each, --clock-control none, bf16, 1 B200)",
           "# commands: tests/probe/run_layer.py / capture_ops.py under ncu --set full -k regex:<kernels>",
           "# (cache control on: cold L2; shares/stalls matter, not the absolute time)", ""]
    traffic = {}
    for name, f, row, desc in CAPS:
        path = os.path.join(PROF, f)
        if not os.path.exists(path):
            continue
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r = list(csv.reader(raw.splitlines()))
        h, u, v = r[0], r[1], r[2 + row]
        out.append("[%s]  (profiles/%s)  %s" % (name, f, desc))
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append("  %-80s %s %s" % (k, v[i], u[i]))
                d[k] = (float(v[i].replace(",", "")), u[i])
        tb = int(d["dram__bytes_read.sum"][0] * SCALE[d["dram__bytes_read.sum"][1]] +
                 d["dram__bytes_write.sum"][0] * SCALE[d["dram__bytes_write.sum"][1]])
        traffic[name] = tb
        out.append("  %-80s %d" % ("dram read+write bytes per launch", tb))
        out.append("")
    open(os.path.join(PROF, "r1_ncu_full_summary.txt"), "w").write("\n".join(out) + "\n")
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from the ncu --set full "
                        "captures in profiles/ (tests/probe/profile_summary.py)")
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)


def launches():
    rows = [r for r in csv.reader(open(os.path.join(PROF, "r1_stack_launches.csv"))) if len(r) > 5]
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
    out = ["# r1 launch list: ncu --metrics gpu__time_duration.sum --clock-control none",
           "# command: python bench.py --steps 3 --warmup 3 --no-cpu-baseline (eager warm-up steps, graph capture,",
           "#          graph replays, L2 flush fills); ncu times are cold-cache and serialised: compare SHARES",
           "launches %d, total %.1f us" % (len(data), tot / 1e3)]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("%-22s n=%4d total=%9.1f us share=%5.1f%% avg=%7.1f us" % (k, n, t / 1e3, 100 * t / tot, t / n / 1e3))
    open(os.path.join(PROF, "r1_stack_launches_summary.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    full_summaries()
    launches()
