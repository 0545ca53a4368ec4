mkdir -p gpurun_out/s8
cap() {  # name, env..., args
  name=$1; shift
  env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:gm4_reg -s 1 -c 1 -o /tmp/$name python tools/ncu_one.py --m 4 --R 1 --B 128 --n $N > gpurun_out/s8/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/s8/$name.raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/s8/$name.details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/s8/$name.source.csv 2>&1
  gzip -f gpurun_out/s8/$name.source.csv
}
N=268435456 cap m4pf TCR_X=0
N=268435456 cap m4nopf TCR_GM_NAT_ALT=9
N=1073741824 cap m4nopf30 TCR_GM_NAT_ALT=9
ls -la gpurun_out/s8
