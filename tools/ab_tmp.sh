for W in cfg3 cfg5; do
for n in cur8 dw1 dw2; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
