for W in cfg4 cfg2; do
for n in nopair pair; do W=$W timeout 300 bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
