"""Print the key metrics of ncu --page raw --csv exports (one line per kernel launch)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "l2rdmiss_sec"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "l2->l1"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
]


def main(paths):
    for p in paths:
        rows = list(csv.reader(open(p)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            print(p.split("/")[-1], r[hdr.index("Kernel Name")][:60])
            out = []
            for k, name in KEYS:
                if k in hdr:
                    out.append(f"{name}={r[hdr.index(k)]}{units[hdr.index(k)] if units[hdr.index(k)] not in ('%', 'inst', '') else ''}")
            print("   ", " ".join(out))
            st = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                    try:
                        st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("    stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1:])
