# Round-1 closing confirmation: full -m gpu suite, smoke(), N=1 bench line.
python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?" > gpurun_out/final_rc.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_rc.txt
python bench.py --steps 20 --warmup 3 > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?" >> gpurun_out/final_rc.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?" >> gpurun_out/final_rc.txt
echo finished
