mkdir -p gpurun_out/dyn
L=$PWD/paper_2510_15271_b200/variants
for rep in 1 2; do
for v in tree cpw2 cpw8 base; do
  case $v in tree) E="";; cpw2) E="SFM_PCG_CPW=2";; cpw8) E="SFM_PCG_CPW=8";; *) E="SFM_B200_LIB=$L/$v.so";; esac
  echo "env=lib:$v" >> gpurun_out/dyn/env_sweep.log
  env $E timeout 300 python tools/pcg_sweep.py 3 8 1e-8:8 >> gpurun_out/dyn/env_sweep.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or config or sharded or large" 2>&1 | tail -2
