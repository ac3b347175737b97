tag=$1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${tag}_nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo done
