# the drop-in leg alone: build and run scripts/dropin_mapping.cpp at config 3
mkdir -p build gpurun_out
g++ -O2 -std=c++17 -pthread -Iinclude -Iscenegen/include scripts/dropin_mapping.cpp -Lpaper_2602_06991_b200/lib -ltkrender \
    -Lscenegen/lib -ltk_synth -Wl,-rpath,$PWD/paper_2602_06991_b200/lib -Wl,-rpath,$PWD/scenegen/lib -o build/dropin_mapping
build/dropin_mapping ${1:-1000000} 1200 680 512 ${2:-10} > gpurun_out/dropin.json 2> gpurun_out/dropin.time
cat gpurun_out/dropin.json
