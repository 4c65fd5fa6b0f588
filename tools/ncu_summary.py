"""Print the handful of ncu metrics we steer by from a .ncu-rep (read on the CPU box)."""
import csv, subprocess, sys
KEEP = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__waves_per_multiprocessor',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio',
        'smsp__average_warp_latency_issue_stalled_barrier.ratio',
        'smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio',
        'smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_mio_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_lg_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_wait.ratio',
        'smsp__average_warp_latency_issue_stalled_not_selected.ratio',
        'smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio',
        'smsp__average_warp_latency_issue_stalled_no_instruction.ratio',
        'smsp__average_warp_latency_issue_stalled_tex_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_membar.ratio',
        'smsp__average_warp_latency_issue_stalled_drain.ratio',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio']
for path in sys.argv[1:]:
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print('====', path, r[idx['Kernel Name']])
        for k in KEEP:
            if k in idx and r[idx[k]] not in ('', '0'):
                print('   %-90s %s %s' % (k, r[idx[k]], units[idx[k]]))
