python -m pytest tests -m gpu -q --timeout 600 -rf -k "histogram or combine or c1 or c3 or pack" > gpurun_out/gpu_tests22.log 2>&1; echo "tests rc=$?" > gpurun_out/rc22.txt
python tools/combine_bench.py --out gpurun_out/combine_r01.json > gpurun_out/combine.log 2>&1; echo "combine rc=$?" >> gpurun_out/rc22.txt
echo finished
