import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; u = r[1]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
 'lts__t_sector_hit_rate.pct','launch__registers_per_thread','sm__throughput.avg.pct_of_peak_sustained_elapsed',
 'l1tex__throughput.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed',
 'smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum',
 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','lts__t_bytes.sum','lts__t_sectors_srcunit_tex.sum',
 'l1tex__m_xbar2l1tex_read_bytes.sum','sm__cycles_elapsed.avg.per_second','lts__t_sectors.sum']
for row in r[2:]:
    print("==", row[h.index("Kernel Name")][:80] if "Kernel Name" in h else "")
    for w in want:
        if w in h: print(f"  {w:70s} {row[h.index(w)]:>20s} {u[h.index(w)]}")
    st = []
    for i, n in enumerate(h):
        if 'smsp__pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
            try: st.append((float(row[i]), n.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except: pass
    tot = sum(x for x, _ in st) or 1
    print("  stalls:", ", ".join(f"{n} {x/tot:.0%}" for x, n in sorted(st, reverse=True)[:8]))
