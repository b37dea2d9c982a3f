# A/B of the exclusion-row kernels on the C3 bench batch (tools/excl_ab.py), then ncu of the default
python -m pytest tests/test_gpu_parity.py -x -q -k "excl or mdps_batched" 2>&1 | tail -2
python tools/excl_ab.py
PS_ELL_ROW=1 python tools/excl_ab.py
ncu --set full --import-source on --clock-control none -k regex:grid_ell --launch-skip 3 -c 1 -o gpurun_out/ell_cell python tools/excl_ab.py > /dev/null 2>&1
