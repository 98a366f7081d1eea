mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_properties.py -x > gpurun_out/props.log 2>&1; echo "props=$?" > gpurun_out/props_status.txt
