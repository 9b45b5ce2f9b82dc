"""Write profiles/<prefix>_ncu_<name>_details.csv (ncu --page details) and
_key.csv (selected raw metrics) from gpurun_out/prof_<name>.ncu-rep.
Usage: python tools/ncu_summaries.py r01_final score pot stats stream"""
import csv
import io
import subprocess
import sys

KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second"]


def main():
    prefix, names = sys.argv[1], sys.argv[2:]
    for n in names:
        rep = f"gpurun_out/prof_{n}.ncu-rep"
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"],
                             capture_output=True, text=True, check=True).stdout
        open(f"profiles/{prefix}_ncu_{n}_details.csv", "w").write(det)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, vals = rows[0], rows[2]
        d = dict(zip(hdr, vals))
        with open(f"profiles/{prefix}_ncu_{n}_key.csv", "w") as f:
            f.write("metric,value\n")
            f.write(f"kernel,\"{d.get('Kernel Name', '')}\"\n")
            for k in KEYS:
                if k in d:
                    f.write(f"{k},{d[k].replace(',', '')}\n")


if __name__ == "__main__":
    main()
