# Round 2: whole GPU suite with the banded kernel on, smoke, the default bench line, config 2's methods
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02_i_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02_i_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_i_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_i_smoke.log
timeout 600 python bench.py > gpurun_out/r02_i_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r02_i_bench.log
bash scripts/cfg2_methods.sh 5 > gpurun_out/r02_i_cfg2.txt 2>&1
tail -n 25 gpurun_out/r02_i_all.log; tail -n 3 gpurun_out/r02_i_smoke.log; cat gpurun_out/r02_i_cfg2.txt | cut -c1-200
