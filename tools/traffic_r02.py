"""profiles/r02_traffic.json from one `ncu --set full` capture of a C3 frame
(tools/gpu/prof2.sh -> gpurun_out/prof_full.ncu-rep): DRAM bytes read +
written per launch of each frame stage (fft = rows + cols kernels), the
`traffic` field of bench.py's roofline.  Not product code.

    python tools/traffic_r02.py gpurun_out/prof_full.ncu-rep profiles/r02_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

STAGE = {"fft_rows_reg_kernel": "fft", "fft_cols_reg_kernel": "fft", "advect_resident_kernel": "advect",
         "smooth_kernel": "smooth", "compose_kernel": "compose", "inject_kernel": "inject"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3,
        "msecond": 1e3}


def main(rep: str, out: str) -> None:
    metrics = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_l1tex2xbar_write_bytes.sum"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kernels, stages = {}, {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hs::", "").split("<")[0]

        def val(m):
            return float(d[m].replace(",", "")) * UNIT.get(u[m], 1.0)
        rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
        kernels[name] = {"time_us": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
                         "sm_to_l2_write_bytes": val("l1tex__m_l1tex2xbar_write_bytes.sum")}
        if name in STAGE:
            stages[STAGE[name]] = stages.get(STAGE[name], 0.0) + rd + wr
    doc = {"config": "C3", "source": rep.split("/")[-1],
           "note": "ncu --set full --clock-control none, one launch of each kernel of a steady-state C3 frame "
                   "(tools/prof_frame.py); ncu flushes caches before each kernel, so reads are cold-cache "
                   "bytes; stages: dram read + write per launch (fft = rows + cols).  DRAM writes read ~0: "
                   "the 126 MB L2 is write-back and holds every kernel's outputs past its end (the "
                   "write-back happens later, outside the kernel); sm_to_l2_write_bytes is what the "
                   "SMs wrote (stores + reductions)",
           "stages": stages, "kernels": kernels}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
