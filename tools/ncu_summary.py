"""Summaries of ncu outputs for profiles/ (run here, without a GPU).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.txt
    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep > profiles/r01_ncu_full.txt
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    seq = [(r[ki], float(r[vi].replace(",", ""))) for r in data if len(r) > vi]
    # split into steps at each sparse/spixel/dense sketch launch of ours
    starts = [i for i, (k, _) in enumerate(seq) if k.startswith(("cdmd::sparse_rows", "cdmd::spixel_rows",
                                                                 "cdmd::sketch_rademacher", "cdmd::sketch_gaussian"))]
    # a step also starts at a dense sketch only when no rows kernel precedes it
    starts = [i for i in starts if not (i > 0 and i - 1 in starts)]
    print(f"# {len(seq)} kernel launches captured (ncu --metrics gpu__time_duration.sum, "
          f"--clock-control none: cold-cache, serialised; compare SHARES)")
    if len(starts) >= 3:
        # the second sequential step (bench.py runs its sequential steps before the
        # streaming lanes, whose launches interleave)
        a, b = starts[1], starts[2]
        step = seq[a:b]
        print(f"# second sequential step: launches {a}..{b - 1} ({len(step)} launches)")
    else:
        step = seq[starts[-1]:] if starts else seq
        print(f"# step from the last sketch launch ({len(step)} launches)")
    tot = sum(v for _, v in step)
    agg = collections.OrderedDict()
    cnt = collections.Counter()
    for k, v in step:
        name = k.split("(")[0][:90]
        agg[name] = agg.get(name, 0.0) + v
        cnt[name] += 1
    ours = sum(v for k, v in agg.items() if k.startswith(("cdmd::", "void cdmd::")))
    print(f"# step total {tot / 1e3:.3f} us-sum -> {tot / 1e6:.3f} ms; our kernels {ours / tot * 100:.1f} %")
    print(f"{'ms':>9} {'share':>6} {'n':>4}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:9.4f} {v / tot * 100:5.1f}% {cnt[k]:4d}  {k}")


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tc.sum",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            # shared-memory bandwidth (the Gaussian sketch's bound)
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
            "smsp__inst_executed_op_shared_ld.sum"]
    units = rows[1]
    for r in rows[2:]:
        print("kernel:", r[h.index("Kernel Name")][:140])
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"  {w:62s} {r[i]:>16s} {units[i]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
