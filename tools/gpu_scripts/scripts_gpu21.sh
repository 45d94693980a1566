python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; echo "smoke rc=$?" > gpurun_out/rc21.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 3 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "histogram_parity or schedule_parity or pack_parity or lpt_assign or eval_parity" -p no:cacheprovider > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/rc21.txt
echo finished
