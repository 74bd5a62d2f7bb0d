mkdir -p gpurun_out
python tools/zgemm_shapes.py C2 > gpurun_out/shapes_c2.log 2>&1
python tools/zgemm_shapes.py C3 > gpurun_out/shapes_c3.log 2>&1
