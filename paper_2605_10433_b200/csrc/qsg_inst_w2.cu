#define QSG_W 2
#include "qsg_inst.cuh"
