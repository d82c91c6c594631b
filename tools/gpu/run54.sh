for rep in 1 2; do for v in 0 1; do echo "== pdl=$v"; HS_PDL=$v SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
HS_PDL=1 timeout 900 python -m pytest tests -m gpu -q -x -k "scene or parity or output" > gpurun_out/r54.log 2>&1; echo "gpu pdl rc=$?"; tail -1 gpurun_out/r54.log
