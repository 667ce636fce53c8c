for W in cfg3 cfg5; do
for n in cur7 e168 e160; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
