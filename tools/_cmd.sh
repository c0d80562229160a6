mkdir -p gpurun_out/rp
L=$PWD/paper_2510_15271_b200/variants
for rep in 1 2; do
for v in tree base; do
  case $v in tree) E="";; *) E="SFM_B200_LIB=$L/$v.so";; esac
  echo "env=lib:$v" >> gpurun_out/rp/env_sweep.log
  env $E timeout 300 python tools/pcg_sweep.py 3 8 1e-8:8 >> gpurun_out/rp/env_sweep.log 2>&1
done; done
