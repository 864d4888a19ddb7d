"""Summarise an ncu report (raw page) into the metrics we track."""
import csv, subprocess, sys, json

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'sm__maximum_warps_per_active_cycle_pct',
        'smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct',
        'smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct',
        'smsp__warps_issue_stalled_wait_per_warp_active.pct',
        'smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct',
        'smsp__warps_issue_stalled_lg_throttle_per_warp_active.pct',
        'smsp__warps_issue_stalled_no_instruction_per_warp_active.pct',
        'smsp__warps_issue_stalled_not_selected_per_warp_active.pct',
        'smsp__warps_issue_stalled_selected_per_warp_active.pct',
        'smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct',
        'smsp__warps_issue_stalled_barrier_per_warp_active.pct',
        'smsp__warps_issue_stalled_branch_resolving_per_warp_active.pct',
        'smsp__warps_issue_stalled_dispatch_stall_per_warp_active.pct',
        'smsp__warps_issue_stalled_drain_per_warp_active.pct',
        'smsp__warps_issue_stalled_imc_miss_per_warp_active.pct',
        'smsp__warps_issue_stalled_membar_per_warp_active.pct',
        'smsp__warps_issue_stalled_misc_per_warp_active.pct',
        'smsp__warps_issue_stalled_sleeping_per_warp_active.pct',
        'smsp__warps_issue_stalled_tex_throttle_per_warp_active.pct',
        'smsp__cycles_active.avg', 'sm__cycles_elapsed.avg', 'smsp__inst_executed_op_global_ld.sum',
        'derived__memory_l1_wavefronts_shared_excessive', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def summary(path):
    out = subprocess.check_output(['ncu', '-i', path, '--page', 'raw', '--csv'], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {'kernel': r[hdr.index('Kernel Name')].split('(')[0]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = r[i] + ((' ' + units[i]) if units[i] else '')
        res.append(d)
    return res


if __name__ == '__main__':
    for p in sys.argv[1:]:
        for d in summary(p):
            print(json.dumps(d, indent=1))
