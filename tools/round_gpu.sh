# End-of-session GPU evidence: tests, smoke, the bench configs, ncu of the fast kernel.
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 1200 python bench.py --config c3 --streams 0 --lattice 0 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
timeout 1200 python bench.py --config c5 --streams 0 --lattice 0 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
[ "${SKIP_PROF:-0}" = 1 ] || bash tools/prof.sh r2c fast
