#define QSG_W 3
#include "qsg_inst.cuh"
