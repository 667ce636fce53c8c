for W in cfg3 cfg5; do
for n in old new old new; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
