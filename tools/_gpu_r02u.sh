mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02u_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02u_smoke.txt
