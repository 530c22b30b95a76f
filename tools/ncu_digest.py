"""Digest of an ncu raw + source CSV export (tools/ncu_kernels.sh): headline metrics,
stall reasons, top stalled SASS lines.  usage: python tools/ncu_digest.py <dir> <kernel>"""
import csv
import re
import sys


def raw(path):
    rows = list(csv.reader(open(path)))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "local_load_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"]


def main(d, k):
    r = raw(f"{d}/raw_{k}.csv")
    for key in KEYS:
        if key in r:
            print(f"{key:80s} {r[key][0]} {r[key][1]}")
    st = {key: float(v[0].replace(",", "")) for key, v in r.items()
          if re.match(r"smsp__pcsamp_warps_issue_stalled_\w+$", key) and not key.endswith("not_issued")
          and v[0].replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    print("stall samples:", int(tot))
    for key, v in sorted(st.items(), key=lambda t: -t[1])[:8]:
        print(f"  {key.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
    rows = list(csv.reader(open(f"{d}/source_{k}.csv")))
    hdr, data = rows[1], rows[2:]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    tot2 = sum(int(x[i_s]) for x in data if x[i_s].isdigit()) or 1
    top = sorted([(int(x[i_s]), j, x[i_src].strip()) for j, x in enumerate(data) if x[i_s].isdigit()], reverse=True)[:25]
    for s, j, src in top:
        print(f"{s:6d} {100 * s / tot2:5.1f}% {j:5d} {src[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
